# scalar sweeps: parity subset + T1/T2/T4 variants (full update)
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused_amr.py tests/test_gpu_run.py -x -q > gpurun_out/pytest_scalar.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_scalar.log
timeout 900 python tools/bench_variants.py --only T1,T2,T4 2>&1 | grep full_update | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['variant'], round(d['ms_per_step'], 4), 'ms', round(d['cell_updates_per_s']/1e9, 1), 'G/s', round(d['hbm_roofline_frac'], 3))"
