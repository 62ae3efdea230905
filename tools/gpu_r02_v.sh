# idle refinement sweeps: max_refine 3 vs 10; compute-sanitizer on small configs
for w in C2 C4; do for mr in 3 10; do timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --max-refine $mr --no-cpu-baseline > gpurun_out/r02v_bench_${w}_mr$mr.json 2>/dev/null; echo bench $w $mr rc $?; done; done
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_run.py C1,C5b2,tiny_eq > gpurun_out/r02v_memcheck.log 2>&1; echo memcheck rc $?
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_run.py C1,tiny_eq > gpurun_out/r02v_synccheck.log 2>&1; echo synccheck rc $?
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report analysis --print-limit 20 python tools/sanitize_run.py C1 > gpurun_out/r02v_racecheck.log 2>&1; echo racecheck rc $?
