# octree: GPU tests (default + the K = 2 variant), O3 timing (default, K = 2), then one ncu --set full
# capture of k3_step on O3 with the summary
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_octree.py -x -q > gpurun_out/pytest_o3.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_o3.log
FC_LIB_PATH=$PWD/variants/k3k2.so timeout 900 python -m pytest tests/test_gpu_octree.py -x -q > gpurun_out/pytest_k3k2.log 2>&1; echo pytest k2 rc=$?; tail -1 gpurun_out/pytest_k3k2.log
o3() { timeout 300 python tools/bench_o3.py 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  try: d=json.loads(l)
  except Exception: continue
  print(round(d['ms_per_step'],4), round(d['value']/1e9,1))"; }
for rep in 1 2 3; do echo "== default"; o3; echo "== k2"; FC_LIB_PATH=$PWD/variants/k3k2.so o3; done
bash tools/gpu_prof_o3.sh > gpurun_out/o3_ncu.txt 2>&1; cat gpurun_out/o3_ncu.txt
