timeout 900 python -m pytest tests/test_gpu_regular_ring.py -x -q > gpurun_out/pytest_reg.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_reg.log
for r in 1 0 1 0; do echo reg=$r; FC_REGULAR_RING=$r timeout 300 python tools/ws_ab.py 2>&1 | tail -2; done
