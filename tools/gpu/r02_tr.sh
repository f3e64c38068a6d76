O=gpurun_out
FZ_LIB_PATH=ab/libfz_trace.so timeout 600 python tools/slice_trace.py T1 T95 T63 T94 C2 C3t2 > $O/r02tr_trace.log 2>&1
