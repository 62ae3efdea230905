# high-MLP big-supernode sweeps
timeout 900 python -m pytest tests -m gpu -x -q -k "subtree_block or c4_parity or test_solve_parity or schedule_variants or c5_full or hykkt_parity or linv" > gpurun_out/r02w_pytest.log 2>&1; echo pytest rc $?
for w in C4 C5 C2 C3 C6; do timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02w_bench_$w.json 2>/dev/null; echo bench $w rc $?; done
timeout 600 python tools/trace_analyze.py C4 > gpurun_out/r02w_trace_c4.txt 2>&1; echo trace rc $?
