# warp-sweep variants: parity subset per variant (FC_LIB_PATH), then C5 / T3 timing per variant
echo default; timeout 300 python tools/ws_ab.py 2>&1 | tail -2
for v in variants/*.so; do echo $v; FC_LIB_PATH=$v timeout 300 python tools/ws_ab.py 2>&1 | tail -2; done
for v in variants/*.so; do FC_LIB_PATH=$v timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "ws or euler or swe" > gpurun_out/pytest_$(basename $v).log 2>&1; echo $v pytest rc=$?; tail -1 gpurun_out/pytest_$(basename $v).log; done
