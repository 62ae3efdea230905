# round-2 check D: tile kernel v2 (per-tile assembly, 1 CTA/SM) -- tests, trace, bench
timeout 900 python -m pytest tests -m gpu -x -q -k "huge or wide or c4_parity or bearing or acopf10000 or C3" > gpurun_out/r02d_pytest.log 2>&1; echo pytest rc $?
timeout 300 python tools/tile_trace.py C4 --save gpurun_out/r02d_tile_trace_c4.npz > gpurun_out/r02d_tile_trace_c4.txt 2>&1; echo trace rc $?
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02d_bench_c4.json 2> gpurun_out/r02d_bench_c4.err; echo bench c4 rc $?
