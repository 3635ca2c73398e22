# A/B of scalar-sweep builds on T1 (quad path and FC_CV_QUAD=0) and T2: default, variants/*.so
for v in default $(ls variants/*.so | xargs -n1 basename | sed 's/\.so$//'); do
  if [ $v = default ]; then unset FC_LIB_PATH; else export FC_LIB_PATH=$PWD/variants/$v.so; fi
  for q in 1 0; do echo "== $v FC_CV_QUAD=$q"; FC_CV_QUAD=$q python tools/bench_variants.py --only T1,T2 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  try: d=json.loads(l)
  except Exception: continue
  if d['mode']=='full_update': print(d['variant'], round(d['ms_per_step'],4))"; done
done
