python tools/trace.py --workload c3_gla2_q2 --ns 3 2>&1 | tail -30
TRACE_RAW=1 TRACE_CTA=5 TRACE_TO=14 python tools/trace.py --workload c3_gla2_q2 --ns 3 2>&1 | tail -15
python tools/trace.py --workload c2_gla2 --ns 2 2>&1 | tail -30
