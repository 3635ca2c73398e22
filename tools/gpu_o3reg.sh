# octree step A/B: O3 timing on the default build and the variants/k3*.so builds, twice each;
# then the octree GPU tests on the default and each variant
python -c "import __graft_entry__ as g; g.build()"
o3() { timeout 300 python tools/bench_o3.py 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  try: d=json.loads(l)
  except Exception: print(l.rstrip()[-200:]); continue
  print(round(d['ms_per_step'],4), round(d['value']/1e9,1))" | tail -3; }
for rep in 1 2; do
  echo "== default"; o3
  for v in variants/k3*.so; do echo "== $v"; FC_LIB_PATH=$PWD/$v o3; done
done
timeout 900 python -m pytest tests/test_gpu_octree.py -x -q > gpurun_out/pytest_o3.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_o3.log
for v in variants/k3*.so; do
  FC_LIB_PATH=$PWD/$v timeout 900 python -m pytest tests/test_gpu_octree.py -x -q > gpurun_out/pytest_$(basename $v .so).log 2>&1; echo pytest $v rc=$?; tail -1 gpurun_out/pytest_$(basename $v .so).log
done
