for c in C1 C2 C5; do timeout 60 python tools/pdl_debug.py $c 2>&1 | tail -1; done
timeout 400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for c in C2 C3 C5 C4; do timeout 120 python bench.py --workload $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; python tools/bench_summary.py gpurun_out/bench_$c.json; tail -1 gpurun_out/bench_$c.err; done
KKT_NO_LINV=1 timeout 120 python bench.py --workload C2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_nolinv.json 2>/dev/null; python tools/bench_summary.py gpurun_out/bench_nolinv.json
KKT_TRACE=1 KKT_NO_GRAPH=1 timeout 120 python tools/trace_analyze.py C2 > gpurun_out/trace_c2.txt 2>&1; grep "==" gpurun_out/trace_c2.txt; python tools/trace_phases.py gpurun_out/trace_raw_C2.npy C2
