# systems kernels: C5 / T3 timing twice, then the systems parity subset
timeout 300 python tools/ws_ab.py 2>&1 | tail -2
timeout 300 python tools/ws_ab.py 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_wsq.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_wsq.log
