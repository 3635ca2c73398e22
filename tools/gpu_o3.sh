# octree step: O3 timing on the default build and each variants/*.so, then the octree parity tests
echo default; timeout 300 python tools/bench_o3.py 2>&1 | tail -1
for v in variants/*.so; do echo $v; FC_LIB_PATH=$v timeout 300 python tools/bench_o3.py 2>&1 | tail -1; done
timeout 900 python -m pytest tests/test_gpu_octree.py -x -q > gpurun_out/pytest_o3.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_o3.log
