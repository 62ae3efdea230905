for c in C4 C6 C2; do timeout 300 python tools/cmp_lib.py $c oldtree 2>&1 | tail -1; done
timeout 600 python -m pytest tests/test_gpu_configs.py -m gpu -x -q -k "tile_solve or subtree or c4_parity or bearing or hykkt_C3" > gpurun_out/pp_pytest.log 2>&1; echo pytest rc $?; tail -1 gpurun_out/pp_pytest.log
for w in C4 C3 C6; do timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/pp_$w.json 2>/dev/null; echo "$w $(python -c "import json;d=json.load(open('gpurun_out/pp_$w.json'));print(round(d['value'],3),d['phases_ms'])")"; done
