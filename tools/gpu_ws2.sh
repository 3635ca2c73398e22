# warp-sweep kernel: parity subset + A/B timing of C5 / T3
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused_amr.py tests/test_gpu_sharded.py -x -q > gpurun_out/pytest_ws.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_ws.log
timeout 300 python tools/ws_ab.py 2>&1 | tail -2
