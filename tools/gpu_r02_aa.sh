# pivot checks off the Cholesky chains
timeout 900 python -m pytest tests -m gpu -x -q -k "not_spd or fail or breakdown or c4_parity or test_solve_parity or huge or ldlt or inertia or c5_full" > gpurun_out/r02aa_pytest.log 2>&1; echo pytest rc $?
for w in C4 C2 C5 C6; do timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02aa_bench_$w.json 2>/dev/null; echo bench $w rc $?; done
