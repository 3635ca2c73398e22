# default build: C5 / T3 timing, then the parity tests that cover every kernel touched by solvers.cuh
timeout 300 python tools/ws_ab.py 2>&1 | tail -2
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hlle.py tests/test_gpu_fused_amr.py tests/test_gpu_full_size.py tests/test_gpu_run.py -x -q > gpurun_out/pytest_ws5.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_ws5.log
