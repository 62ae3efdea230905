# CTA-size selection, C3 with the tile path, ncu of the tree kernels
timeout 900 python -m pytest tests -m gpu -x -q -k "subtree_block or c4_parity or test_solve_parity or c5_full or hykkt" > gpurun_out/r02p_pytest.log 2>&1; echo pytest rc $?
for w in C4 C5 C2 C1 C3 C6; do timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02p_bench_$w.json 2>/dev/null; echo bench $w rc $?; done
KKT_HUGE_SOLVE=1 timeout 300 python bench.py --workload C3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02p_bench_C3_tile.json 2>/dev/null; echo bench C3 tile rc $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tree_ -c 2 -o gpurun_out/r02p_ncu_tree_c4 python bench.py --workload C4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r02p_ncu.log 2>&1; echo ncu rc $?
