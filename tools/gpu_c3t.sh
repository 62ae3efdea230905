KKT_TRACE=1 KKT_NO_GRAPH=1 timeout 120 python tools/trace_analyze.py C3 > gpurun_out/trace_c3.txt 2>&1; grep "==" gpurun_out/trace_c3.txt; python tools/trace_phases.py gpurun_out/trace_raw_C3.npy C3
