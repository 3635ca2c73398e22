timeout 900 python -m pytest tests/test_gpu_octree.py -x -q > gpurun_out/pytest_o3.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_o3.log
for i in 1 2; do timeout 300 python tools/bench_o3.py 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('O3', d['ms_per_step'])"; done
