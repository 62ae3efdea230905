# tree kernels with the CTA view of the large fronts (lite sweeps)
timeout 900 python -m pytest tests -m gpu -x -q -k "subtree_block or hykkt or acopf10000 or huge" > gpurun_out/r02ah_pytest.log 2>&1; echo pytest rc $?
for hs in 0 1; do KKT_HUGE_SOLVE=$hs timeout 300 python bench.py --workload C3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02ah_bench_C3_hs$hs.json 2>/dev/null; echo C3 $hs rc $?; done
for hs in 0 1; do KKT_HUGE_SOLVE=$hs timeout 300 python bench.py --workload C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02ah_bench_C4_hs$hs.json 2>/dev/null; echo C4 $hs rc $?; done
