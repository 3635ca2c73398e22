# round-2 closing verification (second session, after the meta-load changes): smoke, full bench,
# launch list, ncu capture of the headline kernel, full GPU test suite
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -3 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench rc=$?; tail -c 300 gpurun_out/bench_final.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench_final.csv python bench.py --steps 2 --warmup 3 --no-variants --cpu-seconds 0 --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo ncu-launch rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_step_ws -s 3 -c 1 -o gpurun_out/prof_ws_c5_r2d -f python bench.py --steps 2 --warmup 1 --no-variants --cpu-seconds 0 --no-e2e > gpurun_out/ncu_full.log 2>&1; echo ncu-full rc=$?
python tools/ncu_summary.py gpurun_out/prof_ws_c5_r2d.ncu-rep 67108864 > gpurun_out/ws_c5_r2d_ncu.txt 2>&1; cat gpurun_out/ws_c5_r2d_ncu.txt
timeout 2400 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
