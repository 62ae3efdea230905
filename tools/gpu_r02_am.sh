# tile factor trace after the CRIT changes
timeout 300 python tools/tile_trace.py C4 --save gpurun_out/r02am_tile_factor_c4.npz > gpurun_out/r02am_tile_factor_c4.txt 2>&1; echo tf rc $?
for w in C4 C2 C3; do timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02am_bench_$w.json 2>/dev/null; echo $w rc $?; done
