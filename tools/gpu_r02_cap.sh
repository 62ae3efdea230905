for cap in 0 6144 8192 16384 20000; do
  if [ $cap = 0 ]; then E="KKT_X=0"; else E="KKT_SB_CAP=$cap"; fi
  for w in C3 C2; do env $E timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/cap_${cap}_$w.json 2>/dev/null; echo "$cap $w $(python -c "import json;d=json.load(open('gpurun_out/cap_${cap}_$w.json'));print(round(d['value'],3),d['phases_ms']['solve'])" 2>&1 | tail -1)"; done
done
