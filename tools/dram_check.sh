#!/bin/bash
# DRAM bytes of the decode kernel for a workload (ncu, 2 metrics only)
w=$1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:decode_kernel -s 2 -c 1 python tools/prof_step.py --workload $w --steps 3 2>&1 | grep -E "dram__|gpu__time" | sed "s/^/$w /"
