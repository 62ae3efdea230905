# tree-kernel CTA size variants and the block factorisation (opt-in)
for w in C4 C5 C2; do
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02o_bench_$w.json 2>/dev/null; echo bench $w rc $?
  KKT_LIB=paper_2405_14236_b200/libkkt_nt128.so KKT_SB_CAP=4096 timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02o_bench_${w}_nt128.json 2>/dev/null; echo bench nt128 $w rc $?
  KKT_LIB=paper_2405_14236_b200/libkkt_nt128.so KKT_SB_CAP=6144 timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02o_bench_${w}_nt128c6.json 2>/dev/null; echo bench nt128c6 $w rc $?
  KKT_FBLOCK=1 timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02o_bench_${w}_fb.json 2>/dev/null; echo bench fb $w rc $?
done
KKT_LIB=paper_2405_14236_b200/libkkt_nt128.so KKT_SB_CAP=4096 KKT_FBLOCK=1 timeout 600 python tools/trace_analyze.py C4 > gpurun_out/r02o_trace_c4.txt 2>&1; echo trace rc $?
