for r in 1 2 3; do
  echo -n "base "; python bench.py --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],4), d['clocks']['sm_mhz'])"
  echo -n "backoff "; GLAD_LIB=$PWD/abtest/libglad_bo.so python bench.py --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['ms_per_step'],4), d['clocks']['sm_mhz'])"
done
