med() { python -c "import sys,statistics;v=[float(x) for x in sys.stdin.read().split(':')[1].split()];print(round(statistics.median(v[3:]),4))"; }
for w in c3_gla2_q2 c3_gla2_q4; do
 echo -n "base $w "; python tools/abtime.py --workload $w --n 30 | tail -1 | med
 echo -n "rowsNS3 $w "; GLAD_LIB=$PWD/abtest/libglad_NS3.so python tools/abtime.py --workload $w --n 30 | tail -1 | med
done
for w in c2_mla c3_mla_q2 c5_gla8_tp1 c2_gla2_p16 c2_gla2_p1 c1_gla2 c5_gla8_tp8; do
 echo -n "base $w "; python tools/abtime.py --workload $w --n 20 | tail -1 | med
 echo -n "pfall $w "; GLAD_LIB=$PWD/abtest/libglad_pfall.so python tools/abtime.py --workload $w --n 20 | tail -1 | med
done
