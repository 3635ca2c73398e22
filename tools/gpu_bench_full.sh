# full bench (driver contract) + ncu launch list of the same command + one ncu --set full capture of k_step_ws
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo bench rc=$?; tail -c 600 gpurun_out/bench_full.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-variants --cpu-seconds 0 --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo ncu-launch rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_step_ws -s 3 -c 1 -o gpurun_out/prof_ws_c5_full -f python bench.py --steps 2 --warmup 1 --no-variants --cpu-seconds 0 --no-e2e > gpurun_out/ncu_full.log 2>&1; echo ncu-full rc=$?
