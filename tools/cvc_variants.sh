# T4 (and T1 / T2) under tuning builds of the register sweeps, fused and ghost-kernel capacity paths
for v in ${VARIANTS:-default}; do
  if [ $v = default ]; then unset FC_LIB_PATH; else export FC_LIB_PATH=$PWD/variants/$v.so; fi
  for fz in 1 0; do
    echo "== $v fused_capa=$fz"; FC_FUSED_CAPA=$fz python tools/bench_variants.py --only ${ONLY:-T4} 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  try: d=json.loads(l)
  except Exception: continue
  print(d['variant'], d['mode'], round(d['ms_per_step'],4))"
  done
done
