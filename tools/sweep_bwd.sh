for c in 444 296 148 74; do echo "BWD_CTAS $c"; KKT_BWD_CTAS=$c timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err; python tools/bench_summary.py gpurun_out/b.json; tail -1 gpurun_out/b.err; done
timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
