# bench.py under tuning builds of the quiescent copy kernel (VARIANTS="default v256")
for v in ${VARIANTS:-default}; do
  if [ $v = default ]; then unset FC_LIB_PATH; else export FC_LIB_PATH=$PWD/variants/$v.so; fi
  echo "== $v"; python bench.py --cpu-seconds 0 --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value']/1e9,2), round(d['ms_per_step'],4), round(r['launch_ms'],4), round(r['frac'],4))"
done
