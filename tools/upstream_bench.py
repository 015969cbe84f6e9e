"""Time the upstream kernels at the C2 shape (absorb_query, append_rope) with CUDA events."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_21487_b200 import glad
B, Lq, H, d_h, d_c, d_R = 128, 1, 128, 128, 256, 64
dev = "cuda"
qn = torch.randn(B, Lq, H, d_h, device=dev).bfloat16(); qp = torch.randn(B, Lq, H, d_R, device=dev).bfloat16()
w = (torch.randn(H, d_c, d_h, device=dev) / 16).bfloat16(); sl = torch.full((B,), 8192, dtype=torch.int32, device=dev)
out = torch.empty(B, Lq, H, d_c + d_R, dtype=torch.bfloat16, device=dev)
for _ in range(5): glad.gla_absorb_query(qn, qp, w, sl, out=out)
torch.cuda.synchronize()
# device time of the kernel alone: a CUDA graph of 20 launches (no host encode / ctypes cost)
s = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):
        for _ in range(20): glad.gla_absorb_query(qn, qp, w, sl, out=out, stream=s)
torch.cuda.synchronize()
g.replay(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): g.replay()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 200
byts = qn.numel() * 2 + qp.numel() * 2 + w.numel() * 2 + out.numel() * 2
print(f"absorb_query C2 shape: {ms * 1e3:.1f} us, {byts / ms / 1e6:.0f} GB/s algorithmic ({byts / 1e6:.1f} MB)")
