timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --workload C6 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C6.json 2> gpurun_out/bench_C6.err; python tools/bench_summary.py gpurun_out/bench_C6.json; tail -2 gpurun_out/bench_C6.err
KKT_TRACE=1 KKT_NO_GRAPH=1 timeout 600 python tools/trace_analyze.py C6 > gpurun_out/trace_c6.txt 2>&1; grep "==" gpurun_out/trace_c6.txt; sed -n 2,8p gpurun_out/trace_c6.txt
