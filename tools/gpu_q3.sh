timeout 400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
for c in C2 C5 C4 C3; do timeout 150 python bench.py --workload $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; python tools/bench_summary.py gpurun_out/bench_$c.json | cut -c1-150; tail -1 gpurun_out/bench_$c.err; done
