# quad blocks: GPU tests, then T1 timing with and without (FC_CV_QUAD=0)
timeout 900 python -m pytest tests/test_gpu_quad.py tests/test_gpu_parity.py tests/test_gpu_regular_ring.py tests/test_gpu_sharded.py -x -q > gpurun_out/pytest_quad.log 2>&1; echo pytest rc=$?; tail -5 gpurun_out/pytest_quad.log
for q in 1 0 1; do echo "FC_CV_QUAD=$q"; FC_CV_QUAD=$q timeout 300 python tools/bench_variants.py --only T1 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  try: d=json.loads(l)
  except Exception: continue
  print(d['variant'], d['mode'], round(d['ms_per_step'],4), round(d.get('value',0)/1e9,1))"; done
