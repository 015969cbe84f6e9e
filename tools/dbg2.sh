python -m pytest tests -m gpu -x -q 2>&1 | tail -2
tools/sweep.sh c2_gla2:0:7 c3_gla2_q2:0:7 c6_prefill_gla2:0:7
timeout 300 python bench.py --workload c6_prefill_gla2 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline'];print('prefill', d['ms_per_step'], d['tflops'], r['tensor_frac'])"
