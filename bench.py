"""Benchmark: decode attention (GLA-2 / MLA / GTA / GLA-8 TP) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2_gla2] [--impl ours|reference]

One "step" = one pass of the whole hot path (split planning is on the host;
decode kernel + split-KV combine on the device) over one batch of synthetic
input with the BASELINE.json shape.  Default workload is configs[1] (C2,
GLA-2 DeepSeek-V3 shape, B=128, ctx 8K, page 64).

N > 1 (torchrun, one process per GPU, NCCL):
  * c1..c4 workloads: independent decode batches per rank (weak scaling, no
    data-path collective: the problems are independent).
  * c5 workloads: GLA-8 latent heads sharded TP=N: rank r runs
    decode on its h_c/N latent heads and h_q/N query heads, the row-parallel
    o_proj slice (cuBLAS GEMM via torch) and ONE NCCL all-reduce.
Timing: W warm-up steps, then K steps bracketed by barrier + synchronize,
CUDA events on the launching stream, max over ranks.  Rank 0 prints one JSON
line.
"""

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode attention TB/s & TFLOP/s (% B200 roofline); tokens/s at 1/2/4/8 GPUs"


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return dict(hbm=d["hbm_gbs"], bf16=d["bf16_tflops"], bf16_sus=d.get("bf16_tflops_sustained"),
                    src="measured")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, src="fallback")


# ------------------------------------------------------------- oracle leg
def oracle_sample(wl, n_seq=1, seed=0, max_seconds=20.0):
    """Time the fp64 oracle (as it stands) on a bounded sample of `wl`:
    n_seq whole sequences (all heads, all Lq queries) at the workload's
    longest length.  Returns (seconds, tokens, description, threads)."""
    import torch

    import synth
    from oracle import attention as OA

    L = wl.L
    tokens = 0
    t0 = time.perf_counter()
    done = 0
    for s in range(n_seq):
        if wl.variant == "gta":
            q, kv, kr = synth.gta_kernel_inputs(1, wl.Lq, wl.H, wl.h_c, wl.d_c, L, seed=seed + s)
            OA.tied_decode(q, kv, kr, [L], wl.scale, causal=wl.causal)
        else:
            q, c, kr = synth.latent_kernel_inputs(1, wl.Lq, wl.H, wl.h_c, wl.d_c, wl.d_R, L, seed=seed + s)
            OA.latent_decode(q, c, kr, [L], wl.scale, causal=wl.causal)
        tokens += wl.Lq
        done += 1
        if time.perf_counter() - t0 > max_seconds:
            break
    dt = time.perf_counter() - t0
    threads = torch.get_num_threads()
    try:
        import threadpoolctl
        info = threadpoolctl.threadpool_info()
        threads = max([i.get("num_threads", 1) for i in info] + [1])
    except Exception:
        pass
    desc = (f"{done} sequence(s) of ctx {L} x {wl.H} heads x q_len {wl.Lq} ({wl.name} shape), "
            f"fp64 numpy oracle, tokens/s extrapolates linearly in sum(L)*heads")
    return dt, tokens, desc, threads


def run_reference(args, rank):
    """--impl reference: the oracle on the host cores, same metric/unit."""
    from paper_2505_21487_b200 import workloads

    if rank != 0:
        return
    wl = workloads.get(args.workload)
    for _ in range(args.warmup):
        oracle_sample(wl, 1, seed=99, max_seconds=5.0)
    t_total, tok_total = 0.0, 0
    desc, threads = "", 1
    for k in range(args.steps):
        dt, tok, desc, threads = oracle_sample(wl, 1, seed=k, max_seconds=30.0)
        t_total += dt
        tok_total += tok
    # a sampled sequence is at the max length; scale to the workload's mean length
    mean_L = float(np.mean(wl.seqlens()))
    value = tok_total / t_total * (wl.L / mean_L)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_total / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": wl.name, "B": wl.B, "q_len": wl.Lq, "H": wl.H},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": "oracle",
                             "sample": desc},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        smax = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 3 + i and
                          s[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(self.samples)}


# ------------------------------------------------------------- our arm
def _traffic(workload):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get(workload)
    return None


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2505_21487_b200 import glad, tp, workloads

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    name = args.workload
    is_tp = name.startswith("c5")
    if is_tp:
        base = name.replace("_tp1", "").replace("_tp2", "").replace("_tp4", "").replace("_tp8", "")
        name = base.replace("c5_gla8", f"c5_gla8_tp{world}")
    wl = workloads.get(name)
    if args.tile:
        glad.debug_set_tile(args.tile)
    st = workloads.build_device_state(wl, seed=wl.seed + (0 if is_tp else rank), device=dev, num_ctas=args.ctas)
    sl = st["seqlens_host"]
    stream = torch.cuda.current_stream(dev)

    o_proj = None
    if is_tp:  # row-parallel o_proj slice W_r^vo [H_loc*d_c, d_model], d_model 5120 (R15)
        d_model = 5120
        g = torch.Generator(device=dev).manual_seed(1234 + rank)
        w_vo = (torch.randn(wl.H * wl.d_c, d_model, generator=g, device=dev) / math.sqrt(wl.H * wl.d_c)).to(
            torch.bfloat16)
        y = torch.empty(wl.B * wl.Lq, d_model, dtype=torch.bfloat16, device=dev)
        o_proj = (w_vo, y)

    def step():
        out, _ = workloads.run(wl, st, stream=stream)
        if o_proj is not None:  # row-parallel W^vo slice + one all-reduce
            w_vo, y = o_proj
            tp.oproj_allreduce(out.view(wl.B * wl.Lq, wl.H, wl.d_v), w_vo, out=y)
        return out

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize(dev)

    # CUDA graph of one step (host argument marshalling and TMA descriptor
    # encoding happen once at capture; replay is launch-overhead free).
    graph = None
    if not is_tp:
        try:
            g = torch.cuda.CUDAGraph()
            s2 = torch.cuda.Stream(dev)
            s2.wait_stream(stream)
            with torch.cuda.stream(s2):
                with torch.cuda.graph(g, stream=s2):
                    workloads.run(wl, st, stream=s2)
            stream.wait_stream(s2)
            graph = g
            for _ in range(3):
                graph.replay()
            torch.cuda.synchronize(dev)
        except Exception as e:  # eager launches still time the same kernels
            print(f"[bench] graph capture failed ({e}); timing eager launches", file=sys.stderr)
            graph = None

    def timed(fn, K):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(K):
            fn()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        ms = e0.elapsed_time(e1) / K
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    run_step = graph.replay if graph is not None else step
    with ClockSampler(local_rank) as clk:
        t_end = time.perf_counter() + 1.0
        while time.perf_counter() < t_end:  # soak: clocks settle under load
            for _ in range(20):
                run_step()
            torch.cuda.synchronize(dev)
        ms = timed(run_step, args.steps)
    clocks = clk.summary()

    # plan + merge kernels alone (same plan/partials) -> decode kernel share of the step
    glad.debug_set_phase_mask(1 | 4)
    aux_step = lambda: workloads.run(wl, st, stream=stream)
    aux_step()
    aux_ms = timed(aux_step, args.steps)
    glad.debug_set_phase_mask(7)
    decode_ms = max(ms - aux_ms, 1e-9)

    # ---- end to end through the public API with host buffers ----
    pinned_q = st["q"].cpu().pin_memory()
    new_rows = torch.randn(wl.B, wl.Lq, wl.width, generator=torch.Generator().manual_seed(7)).to(
        torch.bfloat16).pin_memory()
    out_h = torch.empty(wl.B, wl.Lq, wl.H, wl.d_v, dtype=torch.bfloat16).pin_memory()
    lse_h = torch.empty(wl.B, wl.Lq, wl.H, dtype=torch.float32).pin_memory()
    q_d = torch.empty_like(st["q"])
    rows_d = torch.empty(wl.B, wl.Lq, wl.width, dtype=torch.bfloat16, device=dev)
    before = (st["seqlens"] - wl.Lq).clamp_min(0).to(torch.int32)

    def e2e_step():
        q_d.copy_(pinned_q, non_blocking=True)
        rows_d.copy_(new_rows, non_blocking=True)
        glad.cache_append(st["layout"], st["pool"], st["block_table"], before, rows_d, stream=stream)
        out, lse = workloads.run(wl, st, stream=stream, q=q_d)
        if o_proj is not None:
            w_vo, y = o_proj
            tp.oproj_allreduce(out.view(wl.B * wl.Lq, wl.H, wl.d_v), w_vo, out=y)
        out_h.copy_(out, non_blocking=True)
        lse_h.copy_(lse, non_blocking=True)

    for _ in range(3):
        e2e_step()
    e2e_ms = timed(e2e_step, args.steps)
    h2d = pinned_q.numel() * 2 + new_rows.numel() * 2
    d2h = out_h.numel() * 2 + lse_h.numel() * 4

    tokens_per_rank = wl.B * wl.Lq
    total_tokens = tokens_per_rank if is_tp else tokens_per_rank * world
    value = total_tokens / (ms * 1e-3)
    abytes = workloads.algorithmic_bytes(wl, sl)
    aflops = workloads.algorithmic_flops(wl, sl)
    pk = _peaks()
    gbs = abytes / (decode_ms * 1e-3) / 1e9
    tfs = aflops / (decode_ms * 1e-3) / 1e12
    hbm_frac = gbs / pk["hbm"]
    ten_frac = tfs / pk["bf16"]
    bound = "hbm" if aflops / abytes < pk["bf16"] * 1e12 / (pk["hbm"] * 1e9) else "tensor"
    roof = {"bound": bound, "achieved": gbs if bound == "hbm" else tfs,
            "peak": pk["hbm"] if bound == "hbm" else pk["bf16"], "unit": "GB/s" if bound == "hbm" else "TFLOP/s",
            "frac": hbm_frac if bound == "hbm" else ten_frac, "traffic": _traffic(wl.name),
            "peak_source": pk["src"] + " (MEASURED_PEAKS.json)",
            "kernel": "glad::decode_kernel", "kernel_ms": decode_ms, "plan_merge_ms": aux_ms,
            "algorithmic_bytes": abytes, "algorithmic_flops": aflops,
            "hbm_frac": hbm_frac, "tensor_frac": ten_frac}
    launches_per_step = 3  # plan, decode, merge

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            dt, tok, desc, threads = oracle_sample(wl, 1, seed=0, max_seconds=20.0)
            mean_L = float(np.mean(sl))
            cpu_val = tok / dt * (wl.L / mean_L)
            cpu = {"value": cpu_val, "unit": "tokens/s", "cores": threads, "kind": "oracle", "sample": desc}
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if is_tp else "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": wl.name, "desc": wl.description, "B": wl.B, "q_len": wl.Lq, "H": wl.H,
                       "n_kv_heads": wl.h_c, "d_head": wl.d_c, "d_rope": wl.d_R, "ctx_max": wl.L,
                       "ctx_mean": float(np.mean(sl)), "page": wl.page, "num_ctas": st["num_ctas"] or "num_SMs",
                       "parallelism": (f"tp{world}" if is_tp else f"dp{world} (independent batches)"),
                       "l2": f"inputs larger than L2 ({abytes / 1e9:.2f} GB algorithmic per step > 126 MB); "
                             "no flush", "cuda_graph": graph is not None},
            "tbps": gbs / 1e3, "tflops": tfs,
            "roofline": roof, "cpu_baseline": cpu,
            "e2e": {"value": total_tokens / (e2e_ms * 1e-3), "unit": "tokens/s", "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "includes": "H2D q + new KV rows (pinned), cache append, plan+decode+merge, D2H out + lse"},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="c2_gla2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ctas", type=int, default=0, help="persistent CTA count (0 = one per SM)")
    ap.add_argument("--tile", type=int, default=0, help="debug: force the KV tile height (0 = library choice)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    import torch.distributed as dist

    if world > 1:
        import torch

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
