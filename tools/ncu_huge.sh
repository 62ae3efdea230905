for k in factor_huge_kernel solve_huge_kernel; do
  KKT_NO_GRAPH=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -s 1 -c 1 -o gpurun_out/prof_c6_$k python tools/run_once.py C6 2 > gpurun_out/ncu_c6_$k.log 2>&1; echo $k rc $?
  ncu -i gpurun_out/prof_c6_$k.ncu-rep --page source --csv --print-source=sass > gpurun_out/src_c6_$k.csv 2>/dev/null
  ncu -i gpurun_out/prof_c6_$k.ncu-rep --page raw --csv > gpurun_out/raw_c6_$k.csv 2>/dev/null
done
