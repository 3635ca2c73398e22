# warp-sweep kernel: parity subset, then A/B timing
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_run.py tests/test_gpu_sharded.py -x -q > gpurun_out/pytest_ws.log 2>&1; echo pytest rc=$?; tail -4 gpurun_out/pytest_ws.log
FC_WS=0 timeout 300 python tools/ws_ab.py 2>&1 | tail -2
timeout 300 python tools/ws_ab.py 2>&1 | tail -2
for v in variants/*.so; do echo $v; FC_LIB_PATH=$v timeout 300 python tools/ws_ab.py 2>&1 | tail -2; done
