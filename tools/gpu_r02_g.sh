# round-2 check G: tile-task solves through the huge fronts
timeout 1500 python -m pytest tests -m gpu -x -q -k "huge or wide or c4_parity or bearing or elec or acopf10000 or ldlt or warp_residual" > gpurun_out/r02g_pytest.log 2>&1; echo pytest rc $?
for w in C4 C6 C7; do timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02g_bench_$w.json 2> gpurun_out/r02g_bench_$w.err; echo bench $w rc $?; done
