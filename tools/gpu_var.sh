timeout 400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
for c in C1 C2 C5 C4; do timeout 120 python bench.py --workload $c --steps 15 --warmup 5 --no-cpu-baseline > gpurun_out/w.json 2>/dev/null; python tools/bench_summary.py gpurun_out/w.json | cut -c1-120; done
