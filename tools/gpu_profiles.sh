set -x
mkdir -p gpurun_out
for w in c2_gla2 c3_gla2_q2 c4_gta; do bash tools/profile_round.sh $w; done
python bench.py --steps 30 --warmup 5 > gpurun_out/bench_c2.json 2>gpurun_out/bench_c2.err
for w in c3_gla2_q2 c3_gla2_q4 c4_gta c2_mla c3_mla_q2 c5_gla8_tp1 c5_gla8_tp8 c2_gla2_p16 c2_gla2_p1; do
  python bench.py --steps 20 --warmup 3 --no-cpu-baseline --workload $w > gpurun_out/bench_$w.json 2>>gpurun_out/bench_all.err
done
ls -la gpurun_out | tail -30
