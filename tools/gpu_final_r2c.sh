# round-2 closing cycle (second session): smoke, full bench, launch list of the same command, ncu
# captures of the headline kernel (C5 k_step_ws) and of the quad-block scalar sweep (T1), full GPU
# test suite
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -3 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench rc=$?; tail -c 300 gpurun_out/bench_final.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench_final.csv python bench.py --steps 2 --warmup 3 --no-variants --cpu-seconds 0 --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo ncu-launch rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_step_ws -s 3 -c 1 -o gpurun_out/prof_ws_c5_r2c -f python bench.py --steps 2 --warmup 1 --no-variants --cpu-seconds 0 --no-e2e > gpurun_out/ncu_full.log 2>&1; echo ncu-full rc=$?
python tools/ncu_summary.py gpurun_out/prof_ws_c5_r2c.ncu-rep 67108864 > gpurun_out/ws_c5_r2c_ncu.txt 2>&1; cat gpurun_out/ws_c5_r2c_ncu.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_step_cv -s 2 -c 1 -o gpurun_out/prof_cv_t1_quad -f python tools/prof_step.py --config C1 --level 10 --m 8 --steps 4 --skip 0 > gpurun_out/ncu_cv_t1.log 2>&1; echo ncu-cv rc=$?
python tools/ncu_summary.py gpurun_out/prof_cv_t1_quad.ncu-rep 67108864 > gpurun_out/cv_t1_quad_ncu.txt 2>&1; cat gpurun_out/cv_t1_quad_ncu.txt
timeout 2400 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
