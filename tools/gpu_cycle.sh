# standard GPU cycle: tests + C5/C3 bench summary
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
for wl in C5 C3; do timeout 400 python bench.py --cpu-seconds 0 --no-e2e --workload $wl > gpurun_out/bench_$wl.log 2>&1; echo bench $wl rc=$?; tail -1 gpurun_out/bench_$wl.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e9,2), round(d['value_full_update']/1e9,3), {k: round(v,4) for k,v in d['phase_ms_per_step'].items()}, d['clocks']['sm_mhz'])"; done
