# k1_memo phase timelines (per-CTA work)
O=gpurun_out
FZ_TRACE_CTAS=1 FZ_SCAN_LG=5 timeout 200 python tools/k1_trace.py C2 C3t3 > $O/k1_trace2.log 2>&1
