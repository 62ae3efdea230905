# chain tasks: two warps per tile, wave size
timeout 900 python -m pytest tests -m gpu -x -q -k "c4_parity or huge or bearing_800 or hykkt_parity or acopf10000 or elec" > gpurun_out/r02y_pytest.log 2>&1; echo pytest rc $?
for wv in 2 3 4; do for w in C4 C6; do KKT_TS_WAVE=$wv timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02y_bench_${w}_w$wv.json 2>/dev/null; echo bench $w $wv rc $?; done; done
