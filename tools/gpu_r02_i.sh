# C4 traces: per-supernode factor/forward/backward + tile-task factor/solve timelines
timeout 600 python tools/trace_analyze.py C4 --json gpurun_out/r02i_trace_c4.json > gpurun_out/r02i_trace_c4.txt 2>&1; echo trace rc $?
timeout 300 python tools/tile_trace.py C4 > gpurun_out/r02i_tile_factor_c4.txt 2>&1; echo tf rc $?
timeout 300 python tools/tile_trace.py C4 --solve > gpurun_out/r02i_tile_solve_c4.txt 2>&1; echo ts rc $?
