set -x
timeout 400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for c in C2 C1 C5 C3; do timeout 400 python bench.py --workload $c --steps 20 --warmup 5 --cpu-sample-s 5 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -c 600 gpurun_out/bench_$c.json; tail -2 gpurun_out/bench_$c.err; done
timeout 600 python bench.py --workload C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err; tail -c 600 gpurun_out/bench_C4.json; tail -3 gpurun_out/bench_C4.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref_C2.json 2>&1; tail -c 400 gpurun_out/bench_ref_C2.json
