"""Cycles per tcgen05.mma (M=128, K=16) for the decode kernel's operand layouts."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

# The microbenchmark kernels are not part of libglad.so: built here into
# tools/microbench/libmicrobench.so (nvcc, sm_100a) on first use.
HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "microbench", "libmicrobench.so")
if not os.path.exists(SO):
    import subprocess
    subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                    "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC", "-shared", "-cudart", "static",
                    "-I" + os.path.join(os.path.dirname(HERE), "paper_2505_21487_b200", "csrc"),
                    os.path.join(HERE, "microbench", "microbench.cu"), "-o", SO], check=True)
lib = ctypes.CDLL(SO)
lib.glad_debug_mma_bench.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
out = torch.zeros(3, dtype=torch.int64, device="cuda")
names = {0: "A K-SW128 / B K-SW128 (QK)", 1: "A MN-SW128 / B MN-noswz (PV now)", 2: "A MN-SW128 / B MN-SW128",
         3: "A MN-SW128 / B K-SW128"}
for iters in (1, 2, 2000):
    for w in (0, 1):
        assert lib.glad_debug_mma_bench(w, 64, iters, ctypes.c_void_p(out.data_ptr())) == 0
        torch.cuda.synchronize()
        cyc, cnt, iss = out.tolist()
        print(f"{cnt:6d} MMAs N=64 {names[w]:34s} total {cyc:8d} cycles, issue loop {iss:8d} cycles")
for n in (16, 64, 128):
    for w in range(4):
        assert lib.glad_debug_mma_bench(w, n, 2000, ctypes.c_void_p(out.data_ptr())) == 0
        torch.cuda.synchronize()
        cyc, cnt, iss = out.tolist()
        ideal = max(128, 128) * n / 256
        print(f"N={n:3d} {names[w]:34s} {cyc / cnt:7.1f} cycles/MMA (dense-rate floor {ideal:.0f})")

# completion time of a burst of n MMAs into an idle pipe (one commit at the end)
lib.glad_debug_mma_burst.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
ob = torch.zeros(64, dtype=torch.int64, device="cuda")
for w in (0, 1):
    for gap in (-1, 5000):
        row = []
        for n in (1, 2, 4, 8, 12, 16, 20, 24, 32):
            assert lib.glad_debug_mma_burst(w, n, gap, ctypes.c_void_p(ob.data_ptr())) == 0
            torch.cuda.synchronize()
            v = ob.tolist()
            row.append(f"n={n}:{v[0]}/{v[32 + n - 1]}")
        print(f"burst {'QK' if w == 0 else 'PV'} gap {gap:5d} done/issued: " + " ".join(row))
