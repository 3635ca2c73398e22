for v in ${VARIANTS:-default u0 u1 u2 u1nb1}; do
  if [ $v = default ]; then unset FC_LIB_PATH; else export FC_LIB_PATH=$PWD/variants/$v.so; fi
  echo "== $v"; python tools/bench_variants.py --only T1,T2 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  try: d=json.loads(l)
  except Exception: continue
  print(d['variant'], d['mode'], round(d['ms_per_step'],4))"
done
