# round-2 check B: HyKKT device loop (CG/CR), C3 bench
timeout 1200 python -m pytest tests -m gpu -x -q -k "hykkt or Krylov or krylov" > gpurun_out/r02b_pytest.log 2>&1; echo pytest rc $?
timeout 300 python bench.py --workload C3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02b_bench_c3.json 2> gpurun_out/r02b_bench_c3.err; echo bench c3 rc $?
