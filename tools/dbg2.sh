python tools/trace.py --workload c3_gla2_q2 --ns 4 2>&1 | sed -n 5,12p
TRACE_RAW=1 TRACE_CTA=5 TRACE_FROM=10 TRACE_TO=16 python tools/trace.py --workload c3_gla2_q2 --ns 4 2>&1 | tail -7
