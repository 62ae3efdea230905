for c in C4 C6 C2 C3; do timeout 300 python tools/cmp_lib.py $c oldtree 2>&1 | tail -1; done
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -m gpu -x -q -k "hykkt or k3 or tile_solve or c4_parity" > gpurun_out/cg_pytest.log 2>&1; echo pytest rc $?; tail -1 gpurun_out/cg_pytest.log
for w in C3 C4; do timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/cg_$w.json 2>/dev/null; echo "$w $(python -c "import json;d=json.load(open('gpurun_out/cg_$w.json'));print(round(d['value'],3),d['phases_ms'],d.get('krylov_iters_total'),d['cg_iters'])")"; done
timeout 200 python tools/kernel_times.py C3 --reps 3 > gpurun_out/kt3_C3.txt 2>&1; grep -v -i warn gpurun_out/kt3_C3.txt | head -12
