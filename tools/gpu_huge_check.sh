timeout 300 python -m pytest tests/test_gpu_parity.py -q -x --timeout 120 -k "wide_front or acopf10000 or bearing or not_spd or NOT_SPD" > gpurun_out/pytest_huge.log 2>&1; tail -3 gpurun_out/pytest_huge.log
timeout 120 python tools/run_once.py C6 2; echo run_once rc $?
bash tools/gpu_test_perf.sh
