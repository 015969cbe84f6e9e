"""Read-only and copy HBM bandwidth on this GPU (context for the roofline:
MEASURED_PEAKS.json's hbm_gbs is a copy, read + write bytes)."""
import statistics

import torch

x = torch.empty(2 * 1024 ** 3, dtype=torch.bfloat16, device="cuda").normal_()
y = torch.empty_like(x)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]


def t(fn, n=10):
    out = []
    for _ in range(n):
        ev[0].record()
        fn()
        ev[1].record()
        torch.cuda.synchronize()
        out.append(ev[0].elapsed_time(ev[1]))
    return statistics.median(out[2:])


nb = x.numel() * 2
ms = t(lambda: x.sum(dtype=torch.float32))
print(f"read (x.sum, {nb / 1e9:.1f} GB): {nb / ms / 1e6:.0f} GB/s")
ms = t(lambda: y.copy_(x))
print(f"copy (read + write {2 * nb / 1e9:.1f} GB): {2 * nb / ms / 1e6:.0f} GB/s")
