# default build: C5 / T3 timing (twice, for the spread), then the systems parity tests
timeout 300 python tools/ws_ab.py 2>&1 | tail -2
timeout 300 python tools/ws_ab.py 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_size.py -x -q > gpurun_out/pytest_ws6.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_ws6.log
