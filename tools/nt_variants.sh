for v in ${VARIANTS:-default}; do
  if [ $v = default ]; then unset FC_LIB_PATH; else export FC_LIB_PATH=$PWD/variants/$v.so; fi
  echo "== $v"; python bench.py --steps 20 --warmup 3 --cpu-seconds 0 --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e9, d['value_full_update']/1e9, d['phase_ms_per_step']['update_full'])"
done
