for c in C4 C6 C2; do timeout 300 python tools/cmp_lib.py $c oldtree 2>&1 | tail -1; done
for w in C4 C2 C5; do timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/rs_$w.json 2>/dev/null; echo "$w $(python -c "import json;d=json.load(open('gpurun_out/rs_$w.json'));print(round(d['value'],3),d['phases_ms'])")"; done
timeout 200 python tools/kernel_times.py C4 --reps 3 > gpurun_out/kt4_C4.txt 2>&1; grep -v -i warn gpurun_out/kt4_C4.txt | head -9
