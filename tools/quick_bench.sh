#!/bin/bash
# usage: tools/quick_bench.sh workload...   (prints one summary line per workload)
for w in "$@"; do
  ws=(${w//:/ }); w=${ws[0]}; sp=${ws[1]:-0}; tt=${ws[2]:-0}
  echo -n "[tile $tt] "
  timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --workload $w --ctas $sp --tile $tt 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.readlines()[-1]); r=d['roofline']
print(d['config']['workload'], 'ctas', d['config']['num_ctas'], 'ms', round(d['ms_per_step'],4), 'TB/s', round(d['tbps'],3), 'hbm', round(r['hbm_frac'],3), 'tc', round(r['tensor_frac'],3), 'e2e_ms', round(d['e2e']['ms_per_step'],4))"
done
