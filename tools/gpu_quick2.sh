# gpu tests + C2/C4/C6 bench + C2 trace
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for c in C2 C4 C5 C3; do timeout 300 python bench.py --workload $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; python tools/bench_summary.py gpurun_out/bench_$c.json; tail -1 gpurun_out/bench_$c.err; done
KKT_TRACE=1 KKT_NO_GRAPH=1 timeout 300 python tools/trace_analyze.py C2 > gpurun_out/trace_c2.txt 2>&1; grep "==" gpurun_out/trace_c2.txt
