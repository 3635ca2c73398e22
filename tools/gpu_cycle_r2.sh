nproc; lscpu | grep "Model name"; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -3 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_r2a.log 2>&1; echo bench rc=$?; tail -c 3000 gpurun_out/bench_r2a.log
timeout 2400 python -m pytest tests -m gpu -x -q -s --durations=15 > gpurun_out/pytest_gpu_r2a.log 2>&1; echo pytest rc=$?; tail -30 gpurun_out/pytest_gpu_r2a.log
