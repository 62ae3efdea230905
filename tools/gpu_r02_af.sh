# factor start lists by critical path; SM reserve for the big kernel
timeout 900 python -m pytest tests -m gpu -x -q -k "c4_parity or test_solve_parity or c5_full or batch_parity" > gpurun_out/r02af_pytest.log 2>&1; echo pytest rc $?
for w in C4 C5 C6 C2; do
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02af_bench_$w.json 2>/dev/null; echo $w rc $?
  for r in 8 16; do KKT_FBIG_RESERVE=$r timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02af_bench_${w}_r$r.json 2>/dev/null; echo $w $r rc $?; done
done
