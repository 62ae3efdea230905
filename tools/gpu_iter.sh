# quick iteration: tile bench, huge-path tests, C4/C6 bench, C6 trace
timeout 60 ./tools/tile_bench
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x --timeout 120 -k "wide_front or acopf10000 or bearing or not_spd or NOT_SPD" > gpurun_out/pytest_huge.log 2>&1; tail -1 gpurun_out/pytest_huge.log
for c in C4 C6; do timeout 300 python bench.py --workload $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; python tools/bench_summary.py gpurun_out/bench_$c.json; done
KKT_TRACE=1 KKT_NO_GRAPH=1 timeout 600 python tools/trace_analyze.py C6 > gpurun_out/trace_c6.txt 2>&1; grep "==" gpurun_out/trace_c6.txt | head -1
