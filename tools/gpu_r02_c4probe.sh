# round-2 C4 probe: trace of factor/forward/backward, ncu launch list of two bench steps, bench line
KKT_TRACE=1 KKT_NO_GRAPH=1 timeout 300 python tools/trace_analyze.py C4 > gpurun_out/r02_trace_c4.txt 2>&1; echo trace rc $?
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_ncu_launches_c4.csv python bench.py --workload C4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02_ncu_c4.log 2>&1; echo ncu rc $?
timeout 300 python bench.py --workload C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_c4.json 2> gpurun_out/r02_bench_c4.err; echo bench rc $?
