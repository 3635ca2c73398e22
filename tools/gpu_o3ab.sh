# octree step: O3 timing (twice) on the default build and each variants/*.so, then the octree GPU tests
for v in default $(ls variants/*.so | xargs -n1 basename | sed 's/\.so$//'); do
  if [ $v = default ]; then unset FC_LIB_PATH; else export FC_LIB_PATH=$PWD/variants/$v.so; fi
  for rep in 1 2; do echo "== $v"; timeout 300 python tools/bench_o3.py 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  try: d=json.loads(l)
  except Exception: continue
  print(round(d['ms_per_step'],4), round(d['value']/1e9,1))"; done
done
unset FC_LIB_PATH
timeout 900 python -m pytest tests -m gpu -k "octree or oct3 or fc3" -x -q > gpurun_out/pytest_o3.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_o3.log
