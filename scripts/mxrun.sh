python -c "from paper_2602_10718_b200 import build as b; b.build(out='paper_2602_10718_b200/libsnapmla_trace.so', defines=['SNAPMLA_TRACE'])"
SNAPMLA_LIB=paper_2602_10718_b200/libsnapmla_trace.so timeout 200 python scripts/trace_mx.py 2>&1 | tail -4
