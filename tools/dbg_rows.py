"""Debug: one rows-mode latent decode case (argv: tile ctas lens...)."""
import sys, os, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import synth
from oracle import attention as OA
from paper_2505_21487_b200 import glad
from gpu_side import build_paged, latent_rows, check, DEV
tile, ctas, d_c = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
lens = np.array([int(x) for x in sys.argv[4:]] or [1500, 63, 640])
glad.debug_set_tile(tile)
B, Lq, H, h_c, d_R = len(lens), 2, 128, 2, 64
q, c, kr = synth.latent_kernel_inputs(B, Lq, H, h_c, d_c, d_R, int(lens.max()), seed=41)
layout, pool, bt = build_paged(latent_rows(c, kr), lens, 64, h_c, d_c, d_R, seed=41)
scale = 1 / math.sqrt(192)
print("stages", glad.lib().glad_debug_set_tile if False else "")
out, lse = glad.gla_decode(q.to(DEV), pool, layout, bt, torch.from_numpy(lens.astype(np.int32)).to(DEV), scale, num_ctas=ctas)
torch.cuda.synchronize()
o_ref, lse_ref = OA.latent_decode(q.double().numpy(), c.double().numpy(), kr.double().numpy(), lens, scale)
check(out, lse, o_ref, lse_ref, what=f"T{tile} ctas {ctas} lens {lens}")
print("OK", tile, ctas, lens)
