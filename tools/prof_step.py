"""Run a few eager decode steps of a workload (for ncu / sanitizer runs)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2505_21487_b200 import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c2_gla2")
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--ctas", type=int, default=0)
a = ap.parse_args()
wl = workloads.get(a.workload)
st = workloads.build_device_state(wl, num_ctas=a.ctas)
for _ in range(a.steps):
    workloads.run(wl, st)
torch.cuda.synchronize()
print("done")
