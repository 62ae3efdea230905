# final round measurement: tests, smoke, bench lines (C2 default with cpu baseline), reference arm, ncu evidence
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 300 python bench.py > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err; python tools/bench_summary.py gpurun_out/bench_C2.json; tail -1 gpurun_out/bench_C2.err
for c in C1 C3 C5 C4 C6; do timeout 300 python bench.py --workload $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; python tools/bench_summary.py gpurun_out/bench_$c.json; tail -1 gpurun_out/bench_$c.err; done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_C2.json 2> gpurun_out/bench_ref_C2.err; tail -c 200 gpurun_out/bench_ref_C2.json
KKT_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ncu_launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo launches rc $?
