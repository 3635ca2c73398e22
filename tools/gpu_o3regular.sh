# octree regular rings A/B: the octree GPU tests with and without the computed-source path
# (FC3_REGULAR=0: the per-patch table for every patch), then O3 timing of each, three times
timeout 900 python -m pytest tests/test_gpu_octree.py -x -q > gpurun_out/pytest_o3_regular.log 2>&1; echo pytest regular rc=$?; tail -1 gpurun_out/pytest_o3_regular.log
FC3_REGULAR=0 timeout 900 python -m pytest tests/test_gpu_octree.py -x -q > gpurun_out/pytest_o3_table.log 2>&1; echo pytest table rc=$?; tail -1 gpurun_out/pytest_o3_table.log
o3() { timeout 300 python tools/bench_o3.py 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  try: d=json.loads(l)
  except Exception: continue
  print(round(d['ms_per_step'],4), round(d['value']/1e9,1))"; }
for rep in 1 2 3; do
  echo "== regular"; o3
  echo "== table"; FC3_REGULAR=0 o3
done
