timeout 1200 python -m pytest tests/test_gpu_regular_ring.py tests/test_gpu_parity.py tests/test_gpu_hlle.py tests/test_gpu_subcycle.py tests/test_gpu_sharded.py tests/test_gpu_run.py -x -q > gpurun_out/pytest_reg.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_reg.log
timeout 600 python tools/var_ab.py 2>&1 | grep '^{'
timeout 300 python tools/ws_ab.py 2>&1 | tail -2
