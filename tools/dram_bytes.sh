#!/bin/bash
# usage: tools/dram_bytes.sh workload [mask]  -> decode kernel duration + DRAM bytes (ncu, one launch)
w=${1:-c2_gla2}; m=${2:-7}
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,launch__cluster_size --clock-control none -k regex:decode_kernel -s 3 -c 1 --csv \
  python tools/abtime.py --workload $w --n 2 --mask $m 2>/dev/null | grep -E '^"[0-9]' | awk -F'","' '{print $(NF-2), $NF}' | sed 's/"//g'
