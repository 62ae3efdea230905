# subtree-block solves: bitwise vs per-node kernels, C4 parity, benches
timeout 900 python -m pytest tests -m gpu -x -q -k "subtree_block or c4_parity or test_solve_parity or batch_parity or schedule_variants" > gpurun_out/r02j_pytest.log 2>&1; echo pytest rc $?
for w in C4 C2 C5; do timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02j_bench_$w.json 2> gpurun_out/r02j_bench_$w.err; echo bench $w rc $?; done
KKT_SBLOCK=0 timeout 300 python bench.py --workload C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02j_bench_C4_nosb.json 2>&1; echo nosb rc $?
