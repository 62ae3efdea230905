for lib in default uc1; do
  for w in C4 C3 C6; do
    if [ $lib = default ]; then L="KKT_X=0"; else L="KKT_LIB=paper_2405_14236_b200/libkkt_$lib.so"; fi
    env $L timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/uc_${lib}_$w.json 2>/dev/null
    echo "$lib $w $(python -c "import json;d=json.load(open('gpurun_out/uc_${lib}_$w.json'));print(round(d['value'],3),d['phases_ms']['solve'])" 2>&1 | tail -1)"
  done
done
