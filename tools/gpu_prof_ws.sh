# one ncu --set full capture of the ws kernel on full C5 (bench command), source view exported here
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_step_ws -s 3 -c 1 -o gpurun_out/prof_ws -f python bench.py --steps 2 --warmup 1 --no-variants --cpu-seconds 0 --no-e2e > /dev/null 2>&1; echo ncu rc=$?
ncu -i gpurun_out/prof_ws.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof_ws_src.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/prof_ws.ncu-rep 67108864
