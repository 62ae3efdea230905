# one GPU round: gpu tests, C2/C3/C4 bench, C4 trace summary
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -5 gpurun_out/pytest_gpu.log
for c in C2 C3; do timeout 400 python bench.py --workload $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; python tools/bench_summary.py gpurun_out/bench_$c.json; tail -2 gpurun_out/bench_$c.err; done
timeout 600 python bench.py --workload C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err; python tools/bench_summary.py gpurun_out/bench_C4.json; tail -3 gpurun_out/bench_C4.err
