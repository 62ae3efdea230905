# full GPU suite with the new defaults; C3 bench; ncu source-level captures of the tile kernels (C4)
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/r02q_pytest.log 2>&1; echo pytest rc $?
timeout 300 python bench.py --workload C3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02q_bench_C3.json 2>/dev/null; echo bench C3 rc $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_factor -c 1 -o gpurun_out/r02q_ncu_tilefactor_c4 python bench.py --workload C4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r02q_ncu1.log 2>&1; echo ncu1 rc $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_solve -c 1 -o gpurun_out/r02q_ncu_tilesolve_c4 python bench.py --workload C4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r02q_ncu2.log 2>&1; echo ncu2 rc $?
