for c in C3 C4 C6; do timeout 60 python tools/pdl_debug.py $c 2>&1 | tail -1; done
timeout 500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for c in C3 C4 C6 C2; do timeout 150 python bench.py --workload $c --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; python tools/bench_summary.py gpurun_out/bench_$c.json; tail -1 gpurun_out/bench_$c.err; done
for c in C3 C4; do KKT_HUGE_SOLVE=1 timeout 150 python bench.py --workload $c --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/bench_hs_$c.json 2>/dev/null; echo "HUGE_SOLVE=1"; python tools/bench_summary.py gpurun_out/bench_hs_$c.json; done
