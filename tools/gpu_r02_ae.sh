# follower row solve in the diagonal Cholesky (CRIT, POTRF0)
timeout 900 python -m pytest tests -m gpu -x -q -k "c4_parity or huge or bearing_800 or acopf10000 or elec or not_spd or hykkt_parity" > gpurun_out/r02ae_pytest.log 2>&1; echo pytest rc $?
for w in C4 C6 C3; do timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02ae_bench_$w.json 2>/dev/null; echo bench $w rc $?; done
