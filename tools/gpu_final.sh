set -x
mkdir -p gpurun_out/final
bash tools/profile_round.sh c2_gla2
python bench.py --steps 30 --warmup 5 > gpurun_out/final/bench_c2.json 2>gpurun_out/final/bench_c2.err
for w in c3_gla2_q2 c3_gla2_q4 c4_gta c2_mla c3_mla_q2 c5_gla8_tp1 c2_gla2_p16 c2_gla2_p1 c3_gla2_q2_p1 c1_gla2; do
  python bench.py --steps 20 --warmup 3 --no-cpu-baseline --workload $w > gpurun_out/final/bench_$w.json 2>>gpurun_out/final/bench_all.err
done
python tools/upstream_bench.py > gpurun_out/final/upstream.txt 2>&1
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final/bench_ref.json 2>&1
