# C3 (HyKKT) breakdown: bench with variants, then an ncu launch list of one step
run() { n=$1; shift; env "$@" timeout 300 python bench.py --workload C3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/c3_$n.json 2> gpurun_out/c3_$n.err; echo "$n rc $? $(python -c "import json;d=json.load(open('gpurun_out/c3_$n.json'));print(round(d['value'],3),d['phases_ms'],d['e2e']['value'],d['cg_iters'],d['refine_iters'],d['gpu_launches'])" 2>&1)"; }
run default KKT_X=0
run nt128 KKT_SB_NT=128
run hs0 KKT_HUGE_SOLVE=0
run chain0 KKT_TS_CHAIN=0
run wave2 KKT_TS_WAVE=2
run nopdl KKT_NO_PDL=1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launches.csv python bench.py --workload C3 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu rc $?
