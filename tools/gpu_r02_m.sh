# tree kernels with hi/lo queues + block factorisation
timeout 900 python -m pytest tests -m gpu -x -q -k "subtree_block or c4_parity or test_solve_parity or batch_parity or schedule_variants or c5_full or hykkt_parity or acopf10000" > gpurun_out/r02m_pytest.log 2>&1; echo pytest rc $?
for w in C4 C2 C1 C5; do timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02m_bench_$w.json 2> gpurun_out/r02m_bench_$w.err; echo bench $w rc $?; done
timeout 600 python tools/trace_analyze.py C4 > gpurun_out/r02m_trace_c4.txt 2>&1; echo trace rc $?
