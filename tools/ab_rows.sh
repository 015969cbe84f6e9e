python -m pytest tests/test_gpu_decode.py -x -q -k "rows or c3_full" 2>&1 | tail -3
for w in c3_gla2_q2 c3_gla2_q4; do for r in 1 2; do
 echo -n "new $w "; python tools/abtime.py --workload $w --n 30 | tail -1 | python -c "import sys,statistics;v=[float(x) for x in sys.stdin.read().split(':')[1].split()];print(round(statistics.median(v[3:]),4))"
 echo -n "old $w "; GLAD_LIB=$PWD/abtest/libglad_old.so python tools/abtime.py --workload $w --n 30 | tail -1 | python -c "import sys,statistics;v=[float(x) for x in sys.stdin.read().split(':')[1].split()];print(round(statistics.median(v[3:]),4))"
done; done
python tools/trace.py --workload c3_gla2_q2 --ns 4 2>&1 | sed -n 1,25p
