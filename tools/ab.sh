#!/bin/bash
# usage: tools/ab.sh workload tile reps  -> median per-call ms (graph) of new vs abtest/libglad_old.so, interleaved
w=${1:-c2_gla2}; t=${2:-128}; r=${3:-3}
for i in $(seq $r); do
  echo -n "new "; python tools/abtime.py --workload $w --tile $t --n 30 | tail -1 | python -c "import sys,statistics;v=[float(x) for x in sys.stdin.read().split(':')[1].split()];print(round(statistics.median(v[3:]),4))"
  echo -n "old "; GLAD_LIB=$PWD/abtest/libglad_old.so python tools/abtime.py --workload $w --tile $t --n 30 | tail -1 | python -c "import sys,statistics;v=[float(x) for x in sys.stdin.read().split(':')[1].split()];print(round(statistics.median(v[3:]),4))"
done
