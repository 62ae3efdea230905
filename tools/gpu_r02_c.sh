# round-2 check C: tile-task factorisation of the huge fronts
timeout 900 python -m pytest tests -m gpu -x -q -k "huge or wide or c4_parity or bearing or acopf10000 or C3" > gpurun_out/r02c_pytest.log 2>&1; echo pytest rc $?
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02c_bench_c4.json 2> gpurun_out/r02c_bench_c4.err; echo bench c4 rc $?
KKT_HUGE_OLD=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02c_bench_c4_old.json 2> gpurun_out/r02c_bench_c4_old.err; echo bench c4 old rc $?
timeout 300 python bench.py --workload C6 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02c_bench_c6.json 2> gpurun_out/r02c_bench_c6.err; echo bench c6 rc $?
