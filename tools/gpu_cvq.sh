# scalar sweeps: T1 / T2 / T4 timing, then the scalar parity / quad / regular-ring / sharded tests
python tools/bench_variants.py --only T1,T2,T4 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  try: d=json.loads(l)
  except Exception: continue
  print(d['variant'], d['mode'], round(d['ms_per_step'],4))"
timeout 900 python -m pytest tests/test_gpu_quad.py tests/test_gpu_parity.py tests/test_gpu_regular_ring.py tests/test_gpu_sharded.py tests/test_gpu_fused_amr.py tests/test_gpu_run.py -x -q > gpurun_out/pytest_cvq.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_cvq.log
