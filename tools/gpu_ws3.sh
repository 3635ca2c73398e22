# warp-sweep variants: parity subset on the default build, then C5 / T3 timing per variant
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_ws.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_ws.log
echo default; timeout 300 python tools/ws_ab.py 2>&1 | tail -2
for v in variants/*.so; do echo $v; FC_LIB_PATH=$v timeout 300 python tools/ws_ab.py 2>&1 | tail -2; done
