med() { python -c "import sys,statistics;v=[float(x) for x in sys.stdin.read().split(':')[1].split()];print(round(statistics.median(v[3:]),4))"; }
for w in c2_gla2 c3_gla2_q2 c5_gla8_tp8 c4_gta; do for r in 1 2; do
 echo -n "new $w "; python tools/abtime.py --workload $w --n 30 | tail -1 | med
 echo -n "old $w "; GLAD_LIB=$PWD/abtest/libglad_old.so python tools/abtime.py --workload $w --n 30 | tail -1 | med
done; done
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
