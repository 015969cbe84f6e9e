"""Debug: one rows-mode latent decode case with parts of q zeroed.
argv: tile ctas zero(none|nope|rope) lens..."""
import sys, os, math
R = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, R); sys.path.insert(0, os.path.join(R, "tests"))
import numpy as np, torch
import synth
from oracle import attention as OA
from paper_2505_21487_b200 import glad
from gpu_side import build_paged, latent_rows, DEV
tile, ctas, zero = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
lens = np.array([int(x) for x in sys.argv[4:]] or [1024, 777])
glad.debug_set_tile(tile)
B, Lq, H, h_c, d_c, d_R = len(lens), 2, 128, 2, 256, 64
q, c, kr = synth.latent_kernel_inputs(B, Lq, H, h_c, d_c, d_R, int(lens.max()), seed=41)
if zero == "nope": q[..., :d_c] = 0
if zero == "rope": q[..., d_c:] = 0
layout, pool, bt = build_paged(latent_rows(c, kr), lens, 64, h_c, d_c, d_R, seed=41)
scale = 1 / math.sqrt(192)
out, lse = glad.gla_decode(q.to(DEV), pool, layout, bt, torch.from_numpy(lens.astype(np.int32)).to(DEV), scale, num_ctas=ctas)
torch.cuda.synchronize()
o_ref, lse_ref = OA.latent_decode(q.double().numpy(), c.double().numpy(), kr.double().numpy(), lens, scale)
o = out.double().cpu().numpy(); l = lse.double().cpu().numpy()
e = np.abs(o - o_ref).max(-1)  # [B, Lq, H]
le = np.abs(l - lse_ref)
print(f"zero={zero} T{tile} ctas {ctas}: max err {e.max():.3e}, lse err {le.max():.3e}")
for b in range(B):
    for t in range(Lq):
        print(f"  b{b} t{t}: out err per head-block of 16: " + " ".join(f"{e[b, t, i:i+16].max():.1e}" for i in range(0, H, 16)) +
              f" | lse err max {le[b, t].max():.1e}")
