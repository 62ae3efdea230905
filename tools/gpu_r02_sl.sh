for c in C4 C2; do timeout 300 python tools/cmp_lib.py $c paper_2405_14236_b200/libkkt_old.so 2>&1 | tail -1; done
for lib in default sl0 sl8; do
  for w in C4 C3; do
    if [ $lib = default ]; then L=""; else L="KKT_LIB=paper_2405_14236_b200/libkkt_$lib.so"; fi
    env $L timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/sl_${lib}_$w.json 2>/dev/null
    echo "$lib $w $(python -c "import json;d=json.load(open('gpurun_out/sl_${lib}_$w.json'));print(round(d['value'],3),d['phases_ms'],d['factor_split_ms'])")"
  done
done
