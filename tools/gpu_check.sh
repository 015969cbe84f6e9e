set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 300 python bench.py --steps 30 --warmup 5 2>&1 | tail -2
tools/sweep.sh c3_gla2_q2:128:7 c3_gla2_q2:128:15 c3_gla2_q2:64:7 c3_gla2_q2:64:15 c3_gla2_q2:96:15 c3_gla2_q4:128:7 c3_gla2_q4:128:15 c3_gla2_q4:64:15 c3_mla_q2:64:7 c3_mla_q2:64:15 c2_mla:64:7 c2_mla:64:15 c2_gla2:128:7
