# tuning builds (python -m paper_1308_1472_b200.build --define ... --out variants/X.so), timed on
# the throughput variants: VARIANTS="default X Y" ONLY=T1,T2 bash tools/cv_variants.sh
for v in ${VARIANTS:-default}; do
  if [ $v = default ]; then unset FC_LIB_PATH; else export FC_LIB_PATH=$PWD/variants/$v.so; fi
  echo "== $v"; python tools/bench_variants.py --only ${ONLY:-T1,T2} 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  try: d=json.loads(l)
  except Exception: continue
  print(d['variant'], d['mode'], round(d['ms_per_step'],4))"
done
