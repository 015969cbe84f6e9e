set -x
timeout 600 python -m pytest tests/test_gpu_decode.py -x -q -k "rows or c3_full" 2>&1 | tail -5
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
tools/sweep.sh c3_gla2_q2:0:7 c3_gla2_q2:0:23 c3_gla2_q2:96:7 c3_gla2_q4:0:7 c3_gla2_q4:96:7 c3_gla2_q2_p1:0:7 c2_gla2:0:7
