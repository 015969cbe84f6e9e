for a in "128 1 128 700 300" "128 1 256 129" "128 1 256 200" "96 1 256 700 300"; do
  echo "== $a"; timeout 60 python tools/dbg_rows.py $a 2>&1 | grep -E "OK|watchdog|Error|assert" | head -3
done
timeout 300 compute-sanitizer --tool memcheck python tools/dbg_rows.py 128 1 256 200 2>&1 | grep -v "^=========     Host Frame" | head -40
