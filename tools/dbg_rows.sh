for z in none nope rope; do timeout 60 python tools/dbg_rows.py 64 0 $z 2>&1 | head -1; done
timeout 60 python tools/dbg_rows.py 64 1 none 2>&1 | head -1
