python -m pytest tests -m gpu -x -q 2>&1 | tail -3
tools/sweep.sh c2_gla2_p1:0:7 c2_gla2_p1:0:39 c3_gla2_q2_p1:0:7 c3_gla2_q2_p1:0:39 c2_gla2:0:7
