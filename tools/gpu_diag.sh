# diagnostics: C2/C4 per-supernode traces, WHILE-node solve graph variant, refine caps
KKT_TRACE=1 KKT_NO_GRAPH=1 timeout 300 python tools/trace_analyze.py C2 > gpurun_out/trace_c2.txt 2>&1; grep "==" gpurun_out/trace_c2.txt
KKT_TRACE=1 KKT_NO_GRAPH=1 timeout 300 python tools/trace_analyze.py C4 > gpurun_out/trace_c4.txt 2>&1; grep "==" gpurun_out/trace_c4.txt
python tools/trace_phases.py gpurun_out/trace_raw_C4.npy C4
for v in 0 1; do KKT_SOLVE_WHILE=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bw$v.json 2>/dev/null; echo WHILE=$v; python tools/bench_summary.py gpurun_out/bw$v.json; done
for r in 0 1 2; do timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --max-refine $r > gpurun_out/br$r.json 2>/dev/null; echo maxref=$r; python tools/bench_summary.py gpurun_out/br$r.json; done
KKT_SOLVE_WHILE=1 timeout 300 python bench.py --workload C5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bw_c5.json 2>/dev/null; python tools/bench_summary.py gpurun_out/bw_c5.json
