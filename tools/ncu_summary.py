"""Summarise ncu artefacts into profiles/ (committed evidence).

    python tools/ncu_summary.py --rep gpurun_out/full_c2.ncu-rep --workload c2_gla2 \
        --launches gpurun_out/launches_c2.csv --out profiles/r01_c2_gla2.md

Reads `ncu -i <rep> --page raw --csv` (one kernel) and the launch-list CSV,
writes a markdown summary and merges dram traffic per launch into
profiles/traffic.json (read by bench.py for roofline.traffic).
"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

KEYS = [
    ("gpu__time_duration.sum", "kernel duration (ncu replay, cold-ish)"),
    ("dram__bytes_read.sum", "DRAM bytes read"),
    ("dram__bytes_write.sum", "DRAM bytes written"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active % (occupancy)"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem / CTA"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum", "local (spill) load sectors"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall: long scoreboard"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall: barrier"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall: wait"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock (Hz)"),
]


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def to_bytes(v, u):
    v = float(str(v).replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u, 1)
    return v * scale


def launches(path):
    if not path or not os.path.exists(path):
        return []
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(io.StringIO("".join(lines))))
    hdr = rows[0]
    iname, ival, iunit = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    out = []
    for r in rows[1:]:
        v = float(r[ival].replace(",", ""))
        if r[iunit] == "usecond":
            v *= 1e3
        elif r[iunit] == "msecond":
            v *= 1e6
        out.append((r[iname], v))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", required=True)
    ap.add_argument("--workload", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--out", required=True)
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    m = raw_metrics(a.rep)
    from paper_2505_21487_b200 import workloads
    wl = workloads.get(a.workload)
    sl = wl.seqlens()
    abytes = workloads.algorithmic_bytes(wl, sl)
    lines = [f"# ncu summary — {a.workload} ({wl.description})", "",
             f"Full-set capture of `glad::decode_kernel` (`ncu --set full --clock-control none --import-source on`)."
             f" {a.note}", "", "| metric | value | unit |", "|---|---|---|"]
    for k, label in KEYS:
        if k in m:
            v, u = m[k]
            lines.append(f"| {label} (`{k}`) | {v} | {u} |")
    rd = to_bytes(*m["dram__bytes_read.sum"]) if "dram__bytes_read.sum" in m else None
    wr = to_bytes(*m["dram__bytes_write.sum"]) if "dram__bytes_write.sum" in m else None
    if rd is not None and wr is not None:
        traffic = rd + wr
        lines += ["", f"Algorithmic bytes per launch (SURVEY §8(d)): {abytes:,} B; measured DRAM traffic per launch: "
                  f"{traffic:,.0f} B (ratio {traffic / abytes:.3f})."]
        tp = os.path.join(os.path.dirname(a.out), "traffic.json")
        d = json.load(open(tp)) if os.path.exists(tp) else {}
        d[a.workload] = {"bytes": traffic, "source": os.path.relpath(a.out, os.path.dirname(os.path.dirname(
            os.path.abspath(__file__))))}
        json.dump(d, open(tp, "w"), indent=1, sort_keys=True)
    ls = launches(a.launches)
    if ls:
        tot = sum(v for _, v in ls)
        by = {}
        for n, v in ls:
            key = n.split("(")[0].replace("void ", "")[:70]
            by.setdefault(key, []).append(v)
        lines += ["", f"Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`, {len(ls)} launches, "
                  "cold-cache serialised — compare shares, not absolutes):", "",
                  "| kernel | launches | mean us | share of listed time |", "|---|---|---|---|"]
        for k, vs in sorted(by.items(), key=lambda kv: -sum(kv[1])):
            lines.append(f"| `{k}` | {len(vs)} | {sum(vs) / len(vs) / 1e3:.1f} | {sum(vs) / tot:.1%} |")
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    open(a.out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
