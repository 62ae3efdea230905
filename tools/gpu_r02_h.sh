# round-2 re-entry: full GPU suite, smoke, default bench (C4), per-config bench lines, C4 launch list
timeout 3000 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/r02h_pytest_gpu.log 2>&1; echo pytest rc $?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02h_smoke.log 2>&1; echo smoke rc $?
timeout 600 python bench.py > gpurun_out/r02h_bench_default.json 2> gpurun_out/r02h_bench_default.err; echo bench rc $?
for w in C1 C2 C3 C5 C6 C7; do timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02h_bench_$w.json 2> gpurun_out/r02h_bench_$w.err; echo bench $w rc $?; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02h_ncu_launches_c4.csv python bench.py --workload C4 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu rc $?
