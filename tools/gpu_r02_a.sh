# round-2 check A: GPU tests (all), smoke, C4 + C2 bench lines
timeout 2400 python -m pytest tests -m gpu -x -q --durations=25 > gpurun_out/r02a_pytest.log 2>&1; echo pytest rc $?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02a_smoke.log 2>&1; echo smoke rc $?
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02a_bench_c4.json 2> gpurun_out/r02a_bench_c4.err; echo bench c4 rc $?
timeout 300 python bench.py --workload C2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02a_bench_c2.json 2> gpurun_out/r02a_bench_c2.err; echo bench c2 rc $?
KKT_SOLVE_IF=1 timeout 300 python bench.py --workload C2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02a_bench_c2_if.json 2> gpurun_out/r02a_bench_c2_if.err; echo bench c2 if rc $?
