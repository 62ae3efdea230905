timeout 400 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for v in 1 0; do for c in C2 C1 C5; do KKT_SOLVE_IF=$v timeout 120 python bench.py --workload $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/w.json 2>/dev/null; echo "IF=$v $(python tools/bench_summary.py gpurun_out/w.json | cut -c1-160)"; done; done
