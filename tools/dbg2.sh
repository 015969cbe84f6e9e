med() { python -c "import sys,statistics;v=[float(x) for x in sys.stdin.read().split(':')[1].split()];print(round(statistics.median(v[3:]),4))"; }

for w in c2_gla2 c3_gla2_q2 c3_gla2_q4 c4_gta; do for r in 1 2; do
 echo -n "base $w "; python tools/abtime.py --workload $w --n 30 | tail -1 | med
 echo -n "poly2 $w "; GLAD_LIB=$PWD/abtest/libglad_poly2.so python tools/abtime.py --workload $w --n 30 | tail -1 | med
 echo -n "poly4 $w "; GLAD_LIB=$PWD/abtest/libglad_poly4.so python tools/abtime.py --workload $w --n 30 | tail -1 | med
done; done
GLAD_LIB=$PWD/abtest/libglad_poly4.so python -m pytest tests/test_gpu_decode.py -q -x -k "peaked or rows_mode or gla_sweep" 2>&1 | tail -2
