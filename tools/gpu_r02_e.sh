# round-2 check E: K3 refinement, elec, bearing 800 parity; C7 bench
timeout 1200 python -m pytest tests -m gpu -x -q -k "unreduced or elec or bearing_800" > gpurun_out/r02e_pytest.log 2>&1; echo pytest rc $?
timeout 300 python bench.py --workload C7 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02e_bench_c7.json 2> gpurun_out/r02e_bench_c7.err; echo bench c7 rc $?
