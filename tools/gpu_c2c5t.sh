timeout 400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
for i in 1 2; do for c in C2 C5; do timeout 120 python bench.py --workload $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/w.json 2>/dev/null; python tools/bench_summary.py gpurun_out/w.json | cut -c1-120; done; done
timeout 120 python bench.py --workload C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/w.json 2>/dev/null; python tools/bench_summary.py gpurun_out/w.json | cut -c1-120
