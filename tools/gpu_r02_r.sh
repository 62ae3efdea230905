# tile-solve chain tweaks: parity + bench; tile factor / solve task traces (C4)
timeout 900 python -m pytest tests -m gpu -x -q -k "c4_parity or huge or bearing_800 or hykkt_parity or acopf10000" > gpurun_out/r02r_pytest.log 2>&1; echo pytest rc $?
for w in C4 C3 C6; do timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02r_bench_$w.json 2>/dev/null; echo bench $w rc $?; done
timeout 300 python tools/tile_trace.py C4 --save gpurun_out/r02r_tile_factor_c4.npz > gpurun_out/r02r_tile_factor_c4.txt 2>&1; echo tf rc $?
timeout 300 python tools/tile_trace.py C4 --solve --save gpurun_out/r02r_tile_solve_c4.npz > gpurun_out/r02r_tile_solve_c4.txt 2>&1; echo ts rc $?
KKT_SOLVE_WHILE=1 timeout 300 python bench.py --workload C2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02r_bench_C2_while.json 2>/dev/null; echo while rc $?
timeout 300 python bench.py --workload C2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02r_bench_C2.json 2>/dev/null; echo c2 rc $?
