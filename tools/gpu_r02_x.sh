# tile-solve chains v2 (TMA ring, per-warp tile products): parity with chains on, benches
KKT_TS_CHAIN=1 timeout 900 python -m pytest tests -m gpu -x -q -k "c4_parity or huge or bearing_800 or hykkt_parity or acopf10000 or C3_gamma or elec" > gpurun_out/r02x_pytest.log 2>&1; echo pytest rc $?
for w in C4 C3 C6; do KKT_TS_CHAIN=1 timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02x_bench_${w}_chain.json 2>/dev/null; echo bench $w rc $?; done
KKT_TS_CHAIN=1 timeout 300 python tools/tile_trace.py C4 --solve --save gpurun_out/r02x_tile_solve_c4.npz > gpurun_out/r02x_tile_solve_c4.txt 2>&1; echo ts rc $?
