med() { python -c "import sys,statistics;v=[float(x) for x in sys.stdin.read().split(':')[1].split()];print(round(statistics.median(v[3:]),4))"; }
python -m pytest tests -m gpu -q 2>&1 | tail -2
for w in c3_gla2_q2 c3_gla2_q4 c6_prefill_gla2; do for r in 1 2; do
 echo -n "wg1 $w "; python tools/abtime.py --workload $w --n 20 | tail -1 | med
 echo -n "wg2 $w "; GLAD_LIB=$PWD/abtest/libglad_wg2.so python tools/abtime.py --workload $w --n 20 | tail -1 | med
done; done
