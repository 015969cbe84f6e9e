"""Markdown table of a tools/bench_all.sh run.

    python tools/bench_table.py gpurun_out/bench_all
"""
import glob
import json
import os
import sys


def main(d):
    rows = []
    for f in sorted(glob.glob(os.path.join(d, "*.json"))):
        name = os.path.basename(f)[:-5]
        try:
            j = json.load(open(f))
        except ValueError:
            continue
        r = j.get("roofline")
        if not r:
            continue
        km = r["kernel_ms"]["median"] if isinstance(r.get("kernel_ms"), dict) else r.get("kernel_ms")
        hbm = r.get("hbm_frac")
        tc = r.get("tensor_frac")
        rows.append(f"| {name} | {j['config'].get('desc', '')} | {j['ms_per_step']:.3f} | {km:.3f} | "
                    f"{'' if hbm is None else f'{100 * hbm:.0f} %'} | {'' if tc is None else f'{100 * tc:.0f} %'} | "
                    f"{j['clocks']['sm_mhz']:.0f} | {j['e2e']['ms_per_step']:.3f} |")
    print("| workload | shape | step ms | kernel ms | % HBM | tensor % | SM MHz | e2e ms |")
    print("|---|---|---|---|---|---|---|---|")
    print("\n".join(rows))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/bench_all")
