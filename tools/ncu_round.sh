# ncu evidence for profiles/: launch list of the bench command and full sets of the top kernels
KKT_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ncu_launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo launches rc $?
for k in factor_big_kernel factor_small_kernel bwd_small_kernel fwd_small_kernel; do
  KKT_NO_GRAPH=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 6 -c 1 -o gpurun_out/prof_$k python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_$k.log 2>&1; echo $k rc $?
done
