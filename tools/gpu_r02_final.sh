# round-2 final measurements: GPU suite, smoke, bench lines (C4 default with cpu_baseline, all configs),
# the reference arm, the C4 ncu launch list (-> traffic json) and full-set captures of the top kernels
timeout 3000 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/final_pytest_gpu.log 2>&1; echo pytest rc $?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo smoke rc $?
timeout 900 python bench.py > gpurun_out/final_bench_C4.json 2> gpurun_out/final_bench_C4.err; echo bench rc $?
for w in C1 C2 C3 C5 C6 C7; do timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/final_bench_$w.json 2> gpurun_out/final_bench_$w.err; echo bench $w rc $?; done
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/final_bench_ref_C4.json 2> gpurun_out/final_bench_ref_C4.err; echo ref rc $?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/final_ncu_launches_c4.csv python bench.py --workload C4 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu list rc $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tile_factor|tree_fwd|tree_bwd|tile_solve" -c 4 -o gpurun_out/final_ncu_full_c4 python bench.py --workload C4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/final_ncu_full.log 2>&1; echo ncu full rc $?
