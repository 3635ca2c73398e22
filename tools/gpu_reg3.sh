timeout 900 python -m pytest tests/test_gpu_regular_ring.py tests/test_gpu_parity.py tests/test_gpu_fused_amr.py -x -q > gpurun_out/pytest_reg.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_reg.log
timeout 600 python tools/var_ab.py 2>&1 | grep '^{'
FC_REGULAR_RING=0 timeout 600 python tools/var_ab.py 2>&1 | grep '^{' | head -4
timeout 300 python tools/ws_ab.py 2>&1 | tail -2; FC_REGULAR_RING=0 timeout 300 python tools/ws_ab.py 2>&1 | tail -2
