# full GPU suite + smoke
timeout 3000 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/r02_pytest_gpu.log 2>&1; echo pytest rc $?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo smoke rc $?
