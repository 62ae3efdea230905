timeout 300 ncu --set full --import-source on --clock-control none -k regex:linv -s 3 -c 1 -o gpurun_out/linv_c2 -f python bench.py --workload C2 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu -i gpurun_out/linv_c2.ncu-rep --page details --csv > gpurun_out/linv_c2_details.csv 2>&1
ncu -i gpurun_out/linv_c2.ncu-rep --page source --csv > gpurun_out/linv_c2_source.csv 2>&1
ls -la gpurun_out/linv_c2*
