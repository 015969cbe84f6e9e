med() { python -c "import sys,statistics;v=[float(x) for x in sys.stdin.read().split(':')[1].split()];print(round(statistics.median(v[3:]),4))"; }
python -m pytest tests/test_gpu_decode.py -x -q -k "rows or prefill or peaked or c3_full or seq_split or fused" 2>&1 | tail -2
for w in c3_gla2_q2 c3_gla2_q4 c6_prefill_gla2; do for r in 1 2; do
 echo -n "new $w "; python tools/abtime.py --workload $w --n 20 | tail -1 | med
 echo -n "old $w "; GLAD_LIB=$PWD/abtest/libglad_old.so python tools/abtime.py --workload $w --n 20 | tail -1 | med
done; done
