timeout 60 ./tools/tile_bench | head -2
timeout 300 python tools/root_steps.py C6 > gpurun_out/root_steps.txt 2>&1; sed -n 3,6p gpurun_out/root_steps.txt; tail -1 gpurun_out/root_steps.txt
for c in C4 C6; do timeout 300 python bench.py --workload $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; python tools/bench_summary.py gpurun_out/bench_$c.json; done
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x --timeout 120 -k "wide_front or acopf10000 or bearing or not_spd or NOT_SPD" 2>&1 | tail -1
