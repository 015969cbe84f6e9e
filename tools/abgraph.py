"""A/B timing of library variants (one process per variant, interleaved).

    python tools/abgraph.py --workload c2_gla2 --libs paper_2505_21487_b200/libglad.so abtest/libglad_b.so --reps 3

Each child loads one library (GLAD_LIB) and prints the median over 50 CUDA
graph replays of (a) the decode launch alone (phase mask 2) and (b) the
whole step (plan + decode + merge), as bench.py times them.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def child(a):
    sys.path.insert(0, ROOT)
    import torch

    from paper_2505_21487_b200 import glad, workloads

    if a.tile:
        glad.debug_set_tile(a.tile)
    wl = workloads.get(a.workload)
    st = workloads.build_device_state(wl, num_ctas=a.ctas)
    s = torch.cuda.Stream()

    def graph(mask):
        glad.debug_set_phase_mask(mask)
        with torch.cuda.stream(s):
            for _ in range(3):
                workloads.run(wl, st, stream=s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            workloads.run(wl, st, stream=s)
        glad.debug_set_phase_mask(a.base_mask)
        return g

    def timeit(g, n=50):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
        with torch.cuda.stream(s):
            for _ in range(10):
                g.replay()
            ev[0].record(s)
            for i in range(n):
                g.replay()
                ev[i + 1].record(s)
        torch.cuda.synchronize()
        return statistics.median(ev[i].elapsed_time(ev[i + 1]) for i in range(n))

    glad.debug_set_phase_mask(a.base_mask)
    gs = graph(a.base_mask)
    if a.soak > 0:  # power-capped clock state, as bench.py times it
        import time
        t_end = time.time() + a.soak
        with torch.cuda.stream(s):
            while time.time() < t_end:
                for _ in range(100):
                    gs.replay()
                torch.cuda.synchronize()
    glad.debug_set_phase_mask(1 | (a.base_mask & ~7))
    workloads.run(wl, st, stream=s)
    gd = graph(2 | (a.base_mask & ~7))
    res = {"step": timeit(gs), "decode": timeit(gd)}
    print("RESULT " + json.dumps(res))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2_gla2")
    ap.add_argument("--libs", nargs="+", default=[os.path.join(ROOT, "paper_2505_21487_b200", "libglad.so")])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--tile", type=int, default=0)
    ap.add_argument("--ctas", type=int, default=0)
    ap.add_argument("--base-mask", type=int, default=7)
    ap.add_argument("--soak", type=float, default=0.0, help="seconds of step replays before timing")
    ap.add_argument("--child", action="store_true")
    a = ap.parse_args()
    if a.child:
        child(a)
        return
    out = {lib: {"step": [], "decode": []} for lib in a.libs}
    for _ in range(a.reps):
        for lib in a.libs:
            env = dict(os.environ, GLAD_LIB=os.path.abspath(lib))
            r = subprocess.run([sys.executable, __file__, "--child", "--workload", a.workload, "--tile", str(a.tile),
                                "--ctas", str(a.ctas), "--base-mask", str(a.base_mask), "--soak", str(a.soak)],
                               env=env, capture_output=True, text=True, timeout=600)
            line = [x for x in r.stdout.splitlines() if x.startswith("RESULT ")]
            if not line:
                print(lib, "FAILED", r.stderr[-2000:])
                continue
            d = json.loads(line[0][7:])
            for k in d:
                out[lib][k].append(d[k])
    for lib, d in out.items():
        if d["step"]:
            print(f"{a.workload:16s} {os.path.basename(os.path.dirname(lib)) + '/' + os.path.basename(lib):40s} "
                  f"step {statistics.median(d['step']):.4f} ms  decode {statistics.median(d['decode']):.4f} ms  "
                  f"(decode runs {' '.join(f'{x:.4f}' for x in d['decode'])})")


if __name__ == "__main__":
    main()
