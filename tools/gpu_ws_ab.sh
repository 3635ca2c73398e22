# A/B of the warp-sweep kernel builds: default libfc.so, then each variants/*.so (C5 / T3 full
# update, ms per step, tools/ws_ab.py), default again; then the systems parity subset on the default
echo default; timeout 300 python tools/ws_ab.py 2>&1 | tail -2
for v in variants/*.so; do echo $v; FC_LIB_PATH=$v timeout 300 python tools/ws_ab.py 2>&1 | tail -2; done
echo default; timeout 300 python tools/ws_ab.py 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_wsab.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_wsab.log
