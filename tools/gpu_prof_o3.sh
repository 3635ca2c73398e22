# ncu --set full capture of the octree step kernel on O3 (tools/bench_o3.py), source view exported
timeout 300 python tools/bench_o3.py > /dev/null 2>&1 && timeout 600 ncu --set full --import-source on --clock-control none -k regex:k3_step -s 3 -c 1 -o gpurun_out/prof_o3 -f python tools/bench_o3.py > /dev/null 2>&1; echo o3 rc=$?
ncu -i gpurun_out/prof_o3.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof_o3_src.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/prof_o3.ncu-rep 33554432
