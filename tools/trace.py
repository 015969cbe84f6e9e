"""Per-CTA pipeline timeline of one decode step (debug tracing in the kernel).

    python tools/trace.py --workload c2_gla2 [--splits N]

Prints medians over CTAs of the per-tile stage latencies (ns):
  load->QK   TMA load issued -> QK issued (load latency + MMA queueing)
  QK->S      QK issued -> S seen by softmax (MMA time + signalling)
  S->P       softmax time (S read -> P written)
  P->PV      P written -> PV issued
  PV->load   PV(i) issued -> load(i+NS) issued (PV time + stage release)
  period     QK(i) -> QK(i+1) issue interval
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
# the timeline instrumentation is compiled only into the trace build
if "GLAD_LIB" not in os.environ:
    import subprocess
    so = os.path.join(ROOT, "paper_2505_21487_b200", "libglad_trace.so")
    subprocess.run([sys.executable, "-m", "paper_2505_21487_b200.build"], cwd=ROOT, check=True,
                   env=dict(os.environ, GLAD_EXTRA_FLAGS="-DGLAD_TRACE=1", GLAD_LIB_OUT=so), stdout=subprocess.DEVNULL)
    os.environ["GLAD_LIB"] = so
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2505_21487_b200 import glad, workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c2_gla2")
ap.add_argument("--ctas", type=int, default=0)
ap.add_argument("--tile", type=int, default=0)
ap.add_argument("--ns", type=int, default=2, help="KV stages of the instantiation (for PV->load)")
ap.add_argument("--mask", type=int, default=7, help="glad_debug_set_phase_mask value")
ap.add_argument("--soak", type=float, default=0.0, help="seconds of back-to-back steps before the traced one (power-capped clock)")
a = ap.parse_args()
wl = workloads.get(a.workload)
glad.debug_set_phase_mask(a.mask)
if a.tile:
    glad.debug_set_tile(a.tile)
st = workloads.build_device_state(wl, num_ctas=a.ctas)
for _ in range(3):
    workloads.run(wl, st)
torch.cuda.synchronize()
if a.soak > 0:
    import time
    t_end = time.time() + a.soak
    while time.time() < t_end:
        for _ in range(200):
            workloads.run(wl, st)
        torch.cuda.synchronize()
n_ctas = 70000
buf = torch.zeros(n_ctas * glad.TRACE_STRIDE, dtype=torch.int64, device="cuda")
glad.debug_set_trace(buf)
workloads.run(wl, st)
torch.cuda.synchronize()
glad.debug_set_trace(None)
tr = buf.view(n_ctas, glad.TRACE_STRIDE).cpu().numpy().astype(np.int64)
tr = tr[tr[:, 0] > 0]
t0 = tr[:, 0].min()
print(f"{wl.name}: segments/CTA {np.median(tr[:, 3]):.1f}, {len(tr)} CTAs, kernel span {(tr[:, 2].max() - t0) / 1e3:.1f} us")
_st = np.sort(tr[:, 0] - t0) / 1e3
_en = np.sort(tr[:, 2] - t0) / 1e3
print("CTA start (us, percentiles 0/50/90/100): " + " ".join(f"{np.percentile(_st, q):.1f}" for q in (0, 50, 90, 100)) +
      "; end: " + " ".join(f"{np.percentile(_en, q):.1f}" for q in (0, 10, 50, 90, 100)))
print(f"kernel entry -> CTA start (setup) us: median {np.median(tr[:, 0] - tr[:, 7]) / 1e3:.1f} max {np.max(tr[:, 0] - tr[:, 7]) / 1e3:.1f}; "
      f"entry spread {(tr[:, 7].max() - tr[:, 7].min()) / 1e3:.1f}")
print(f"CTA lifetime median {np.median(tr[:, 2] - tr[:, 0]) / 1e3:.1f} us, start->Q ready "
      f"{np.median(tr[:, 1] - tr[:, 0]) / 1e3:.2f} us")
T = (tr.shape[1] - 8 - 32) // 12
tile = tr[:, 8:8 + 12 * T].reshape(len(tr), T, 12)  # load, qk, s, p, pv, free, p_wg1, epi, qk_ret, pv_ret, landed, -
valid = tile[:, :, 1] > 0
ntile = valid.sum(1)


def med(x, m):
    x = x[m]
    return float(np.median(x)) if x.size else float("nan")


m = valid.copy()
m[:, 0] = False  # skip first tile (pipeline fill)
print("median ns per tile (excluding tile 0):")
print(f"  load->QK  {med(tile[:, :, 1] - tile[:, :, 0], m):8.0f}")
print(f"  QK->S     {med(tile[:, :, 2] - tile[:, :, 1], m):8.0f}")
print(f"  S->P      {med(tile[:, :, 3] - tile[:, :, 2], m):8.0f}")
print(f"  P->PV     {med(tile[:, :, 4] - tile[:, :, 3], m):8.0f}")
print(f"  P(WG1)-P(WG0) {med(tile[:, :, 6] - tile[:, :, 3], m):8.0f}")
print(f"  P(WG1)->PV {med(tile[:, :, 4] - tile[:, :, 6], m):8.0f}")
print(f"  P(last warp)-P(WG0) {med(tile[:, :, 11] - tile[:, :, 3], m & (tile[:, :, 11] > 0)):8.0f}  P(last warp)->PV {med(tile[:, :, 4] - tile[:, :, 11], m & (tile[:, :, 11] > 0)):8.0f}")
ns = a.ns
pv_to_free = tile[:, ns:, 5] - tile[:, :-ns, 4]
print(f"  free(i+{ns})-PV(i) {med(pv_to_free, valid[:, ns:] & valid[:, :-ns]):8.0f}")
print(f"  load-free  {med(tile[:, :, 0] - tile[:, :, 5], m):8.0f}")
pv_to_load = tile[:, :-ns, 4] - tile[:, ns:, 0]
mm = valid[:, ns:] & valid[:, :-ns]
print(f"  load(i+{ns})-PV(i) {med(-pv_to_load, mm):8.0f}")
per = tile[:, 1:, 1] - tile[:, :-1, 1]
print(f"  QK period {med(per, valid[:, 1:] & valid[:, :-1]):8.0f}")
first = tile[:, 0]
print(f"  first tile: start->load {np.median(first[:, 0] - tr[:, 0]):.0f}  load->QK {np.median(first[:, 1] - first[:, 0]):.0f}")
last = np.array([tile[i, ntile[i] - 1, 4] for i in range(len(tr))])
print(f"  last PV issue -> CTA end {np.median(tr[:, 2] - last):.0f}  (tiles traced/CTA {np.median(ntile):.0f})")
# time budget of a median CTA: steady tiles vs segment switches vs start / tail
epi = tile[:, :, 7]
qk = tile[:, :, 1].astype(np.float64)
dq = np.where(valid[:, 1:] & valid[:, :-1], qk[:, 1:] - qk[:, :-1], np.nan)
seg_end = epi[:, :-1] > 0  # tile i ends a segment -> gap to QK(i+1) is a switch
sw = np.where(seg_end, dq, np.nan)
st = np.where(~seg_end, dq, np.nan)
print(f"  per CTA: steady QK->QK sum {np.nanmedian(np.nansum(st, 1)) / 1e3:.1f} us over {np.median(np.sum(~np.isnan(st), 1)):.0f} "
      f"gaps (mean {np.nanmean(st):.0f} ns), switch gaps sum {np.nanmedian(np.nansum(sw, 1)) / 1e3:.1f} us "
      f"(mean {np.nanmean(sw):.0f} ns)")
print(f"  start->first QK {np.median(tr[:, 1] - tr[:, 0]) / 1e3:.1f} us, last QK->end {np.median(tr[:, 2] - np.nanmax(np.where(valid, qk, np.nan), 1)) / 1e3:.1f} us")
print(f"  producer: prefetch cursor ready {np.median(tr[:, -6] - tr[:, 0]) / 1e3:.2f} us after start")
print(f"  start (us): Q issued {np.median(tr[:, 5] - tr[:, 0]) / 1e3:.2f}, producer past Q barrier "
      f"{np.median(tr[:, 4] - tr[:, 0]) / 1e3:.2f}, first row looked up {np.median(tr[:, 6] - tr[:, 0]) / 1e3:.2f}, "
      f"first load issued {np.median(tile[:, 0, 0] - tr[:, 0]) / 1e3:.2f}")
print(f"  epilogue: S(last)->epi done {np.nanmedian(np.where(epi > 0, epi - tile[:, :, 2], np.nan)):.0f} ns")

# end-time spread: which CTAs finish last (segments, tiles, SM id)
_end = (tr[:, 2] - t0) / 1e3
_nseg = tr[:, 3]
print("end time by #segments: " + ", ".join(f"{int(k)} seg: n={int((_nseg == k).sum())} median end "
                                            f"{np.median(_end[_nseg == k]):.1f} us" for k in np.unique(_nseg)))
_ord = np.argsort(_end)[::-1][:8]
print("latest CTAs (end us, start us, #seg, tiles, smid): " + "; ".join(
    f"{_end[i]:.1f} {(tr[i, 0] - t0) / 1e3:.1f} {int(_nseg[i])} {int(ntile[i])} {int(tr[i, -1])}" for i in _ord))
_ord = np.argsort(_end)[:4]
print("earliest CTAs (end us, #seg, tiles, smid): " + "; ".join(
    f"{_end[i]:.1f} {int(_nseg[i])} {int(ntile[i])} {int(tr[i, -1])}" for i in _ord))
_rate = ntile / np.maximum((tr[:, 2] - tr[:, 0]) / 1e3, 1e-9)
print(f"tiles per us over CTAs: min {_rate.min():.3f} p10 {np.percentile(_rate, 10):.3f} median {np.median(_rate):.3f} max {_rate.max():.3f}")

if os.environ.get("TRACE_SWITCH"):
    # raw timelines around the segment switches of the latest 3-seg and an early 2-seg CTA
    picks = [int(np.argsort(_end)[-1]), int(np.argsort(np.where(_nseg == _nseg.min(), _end, 1e18))[len(_end) // 4 % max(1, int((_nseg == _nseg.min()).sum()))])]
    for c in picks:
        base = tr[c, 0]
        print(f"CTA {c} (smid {int(tr[c, -1])}, {int(_nseg[c])} seg, end {_end[c]:.1f} us): tile: free load QK QKret S P0 PV PVret epi nextQ (us)")
        ends = [i for i in range(ntile[c]) if tile[c, i, 7] > 0]
        show = sorted({j for i in ends for j in range(max(0, i - 2), min(ntile[c], i + 4))} | {0, 1, 2, ntile[c] - 1})
        for i in show:
            print(f"  tile {i:3d}: " + "  ".join(f"{(tile[c, i, j] - base) / 1e3:8.2f}" if tile[c, i, j] else "       -"
                                               for j in (5, 0, 1, 8, 2, 3, 4, 9, 7, 10)))

if os.environ.get("TRACE_QSEG"):
    c = int(np.argsort(_end)[-1])
    base = tr[c, 0]
    print(f"CTA {c}: per segment (us): first QK probe, q_full seen, qn_full seen")
    for sg in range(1, 8):
        sl = tr.shape[1] - 32 + 3 * sg
        v = tr[c, sl:sl + 3]
        if v[2]:
            print(f"  seg {sg}: probe {(v[2] - base) / 1e3:8.2f}  q_full {(v[0] - base) / 1e3 if v[0] else -1:8.2f}  "
                  f"qn_full {(v[1] - base) / 1e3 if v[1] else -1:8.2f}")

if os.environ.get("TRACE_RAW"):
    c = int(os.environ.get("TRACE_CTA", "5"))
    base = tr[c, 0]
    print(f"raw timeline of CTA {c} (us from CTA start): free, load, landed, QK, QKret, S, P0, P1, Plast, PV, PVret, epi")
    for i in range(int(os.environ.get("TRACE_FROM", "0")), int(os.environ.get("TRACE_TO", "128"))):
        if tile[c, i, 1] == 0:
            break
        print(f"  tile {i:2d}: " + "  ".join(f"{(tile[c, i, j] - base) / 1e3:8.2f}" if tile[c, i, j] else "       -"
                                          for j in (5, 0, 10, 1, 8, 2, 3, 6, 11, 4, 9, 7)))
