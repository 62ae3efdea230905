# CRIT wait order + no panel copies with the tile solve; chains opt-in
timeout 900 python -m pytest tests -m gpu -x -q -k "c4_parity or huge or bearing_800 or hykkt_parity or acopf10000 or C3_gamma or elec or ldlt" > gpurun_out/r02u_pytest.log 2>&1; echo pytest rc $?
for w in C4 C3 C6; do timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02u_bench_$w.json 2>/dev/null; echo bench $w rc $?; done
KKT_TILE_PANEL=1 timeout 300 python bench.py --workload C4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02u_bench_C4_panel.json 2>/dev/null; echo panel rc $?
