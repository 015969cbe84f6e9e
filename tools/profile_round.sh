#!/bin/bash
# Profiling pass for one workload (run under gpurun, 1 GPU):
#   launch list of the bench command + one full ncu capture of the decode kernel.
w=${1:-c2_gla2}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_$w.csv \
    python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench_$w.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 2 -c 1 \
    -o gpurun_out/full_$w -f python tools/prof_step.py --workload $w --steps 3 > gpurun_out/ncu_full_$w.log 2>&1
echo "profiled $w"
