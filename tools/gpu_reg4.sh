timeout 900 python -m pytest tests/test_gpu_regular_ring.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_reg.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_reg.log
timeout 600 python tools/var_ab.py 2>&1 | grep '^{'
