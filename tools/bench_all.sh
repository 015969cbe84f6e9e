#!/bin/bash
# Bench every workload (run under gpurun, 1 GPU): one JSON line each into
# gpurun_out/bench_all/<workload>.json (the default line carries the CPU baseline).
mkdir -p gpurun_out/bench_all
python bench.py > gpurun_out/bench_all/default_c2_gla2.json 2> gpurun_out/bench_all/default_c2_gla2.err
for w in c1_gla2 c2_mla c2_gla2_p16 c2_gla2_p1 c3_gla2_q2 c3_gla2_q4 c3_mla_q2 c3_gla2_q2_p1 c4_gta \
         c5_gla8_tp1 c5_gla8_tp8 c5_gla8_tp8_skew c6_prefill_gla2 c6_prefill_gla2_mat c7_prefill_gta; do
  timeout 600 python bench.py --workload $w --steps 20 --no-cpu-baseline > gpurun_out/bench_all/$w.json 2> gpurun_out/bench_all/$w.err
done
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_all/reference_c2_gla2.json 2>&1
echo done
