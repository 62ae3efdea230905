for c in C4 C2 C3; do timeout 300 python tools/cmp_lib.py $c oldtree 2>&1 | tail -1; done
for w in C5 C4 C2; do timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/cd_$w.json 2>/dev/null; echo "$w $(python -c "import json;d=json.load(open('gpurun_out/cd_$w.json'));print(round(d['value'],3),d['phases_ms'])")"; done
