# round-2 check F: LDL^T (NEXT-2)
timeout 1500 python -m pytest tests -m gpu -x -q -k "ldlt or inertia" > gpurun_out/r02f_pytest.log 2>&1; echo pytest rc $?
