"""Back-to-back timing of one workload's decode step (eager and CUDA graph)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2505_21487_b200 import glad, workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c2_gla2")
ap.add_argument("--tile", type=int, default=0)
ap.add_argument("--n", type=int, default=20)
ap.add_argument("--trace", action="store_true", help="run with the debug timeline enabled")
ap.add_argument("--mask", type=int, default=7, help="glad_debug_set_phase_mask value")
ap.add_argument("--ctas", type=int, default=0)
a = ap.parse_args()
if a.tile:
    glad.debug_set_tile(a.tile)
glad.debug_set_phase_mask(a.mask)
wl = workloads.get(a.workload)
st = workloads.build_device_state(wl, num_ctas=a.ctas)
if a.trace:
    tbuf = torch.zeros(4096 * glad.TRACE_STRIDE, dtype=torch.int64, device="cuda")
    glad.debug_set_trace(tbuf)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(3):
        workloads.run(wl, st, stream=s)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(a.n + 1)]
with torch.cuda.stream(s):
    ev[0].record(s)
    for i in range(a.n):
        workloads.run(wl, st, stream=s)
        ev[i + 1].record(s)
torch.cuda.synchronize()
print("eager per-call ms:", " ".join(f"{ev[i].elapsed_time(ev[i + 1]):.3f}" for i in range(a.n)))
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    workloads.run(wl, st, stream=s)
torch.cuda.synchronize()
with torch.cuda.stream(s):
    ev[0].record(s)
    for i in range(a.n):
        g.replay()
        ev[i + 1].record(s)
torch.cuda.synchronize()
print("graph per-call ms:", " ".join(f"{ev[i].elapsed_time(ev[i + 1]):.3f}" for i in range(a.n)))
if a.trace:
    import numpy as np
    tr = tbuf.view(4096, glad.TRACE_STRIDE).cpu().numpy().astype(np.int64)
    plan_t = tr[4095, :2].copy()
    tr = tr[:4095]
    tr = tr[tr[:, 0] > 0]
    t0 = tr[:, 7].min()
    print(f"traced CTAs {len(tr)}; entry spread {(tr[:, 7].max() - t0) / 1e3:.1f} us; start max {(tr[:, 0].max() - t0) / 1e3:.1f}; "
          f"end min/med/max {(tr[:, 2].min() - t0) / 1e3:.1f} {(np.median(tr[:, 2]) - t0) / 1e3:.1f} {(tr[:, 2].max() - t0) / 1e3:.1f} us")
    ms_ = tr[:, -4] > 0
    print(f"bg merges: CTAs {ms_.sum()}, start med {(np.median(tr[ms_, -4]) - t0) / 1e3:.1f} us, "
          f"duration med {np.median(tr[ms_, -5] - tr[ms_, -4]) / 1e3:.1f} max {np.max(tr[ms_, -5] - tr[ms_, -4]) / 1e3:.1f} us, "
          f"done max {(tr[ms_, -5].max() - t0) / 1e3:.1f} us")
    w2 = (tr[:, -2] - tr[:, 2]) / 1e3
    print(f"warp 2 reached the end barrier relative to trace[2] (us): min {w2.min():.1f} med {np.median(w2):.1f} max {w2.max():.1f}")
    dd = (tr[:, -1] - tr[:, 2]) / 1e3
    print(f"TMEM dealloc took (us): min {dd.min():.1f} med {np.median(dd):.1f} max {dd.max():.1f}; "
          f"released max {(tr[:, -1].max() - t0) / 1e3:.1f} us")
    print(f"plan kernel: start {(plan_t[0] - t0) / 1e3:.1f} us, end {(plan_t[1] - t0) / 1e3:.1f} us relative to decode entry")
