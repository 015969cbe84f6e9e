cat > /tmp/t.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
from paper_2505_21487_b200 import glad
import test_gpu_decode as T
glad.debug_set_phase_mask(7 | 8 | 64)
for cfg in [(2, 4, 128, 2, 256, 64, [900, 1201], 16, 0, True), (3, 4, 128, 2, 256, 64, [1500, 63, 640], 64, 8, True), (2, 4, 128, 2, 256, 64, [2000, 333], 64, 2, True)]:
    B, Lq, H, h_c, d_c, d_R, lens, page, ctas, causal = cfg
    out, lse, o_ref, lse_ref = T.run_latent(B, Lq, H, h_c, d_c, d_R, np.array(lens), page, ctas=ctas, causal=causal, seed=5)
    try:
        T.check(out, lse, o_ref, lse_ref, what=str(cfg)); print("OK", cfg)
    except AssertionError as e:
        print("FAIL", e)
PY
timeout 120 python /tmp/t.py 2>&1 | tail -4
tools/sweep.sh c3_gla2_q4:0:7 c3_gla2_q4:0:79 c6_prefill_gla2:0:7 c6_prefill_gla2:0:79
