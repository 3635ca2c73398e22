# regular-ring gather: bitwise tests + parity, then variant timing with and without it
timeout 900 python -m pytest tests/test_gpu_regular_ring.py tests/test_gpu_parity.py tests/test_gpu_fused_amr.py -x -q > gpurun_out/pytest_reg.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_reg.log
timeout 600 python tools/var_ab.py 2>&1 | grep '^{'
FC_REGULAR_RING=0 timeout 600 python tools/var_ab.py 2>&1 | grep '^{'
timeout 300 python tools/ws_ab.py 2>&1 | tail -2
