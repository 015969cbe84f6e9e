#!/bin/bash
# usage: tools/sweep.sh "workload:tile:mask ..."  -> median graph ms per config (abtime.py)
for c in $@; do
  ws=(${c//:/ }); w=${ws[0]}; t=${ws[1]:-0}; m=${ws[2]:-7}
  echo -n "$w tile $t mask $m : "
  timeout 300 python tools/abtime.py --workload $w --tile $t --mask $m --n 30 2>&1 | tail -1 | python -c "import sys,statistics;s=sys.stdin.read();v=[float(x) for x in s.split(':')[1].split()] if 'graph' in s else None;print(round(statistics.median(v[3:]),4) if v else s.strip()[-200:])"
done
