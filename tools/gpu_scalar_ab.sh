# scalar sweeps: T1/T2/T4 full update for the default library and every variants/*.so
run() { timeout 900 python tools/bench_variants.py --only T1,T2,T4 2>&1 | grep full_update | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print('  ', d['variant'], round(d['ms_per_step'], 4), 'ms', round(d['cell_updates_per_s']/1e9, 1), 'G/s', round(d['hbm_roofline_frac'], 3))"; }
echo default; run
for v in variants/*.so; do echo $v; FC_LIB_PATH=$v run; done
