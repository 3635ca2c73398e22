# ncu capture of the warp-sweep kernel (C5 physics, level 7, full update)
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_step_ws -s 2 -c 1 -o gpurun_out/prof_ws_c5 -f python tools/prof_step.py --config C5 --level 7 --steps 4 --skip 0 > gpurun_out/ncu_ws.log 2>&1; echo ncu rc=$?; tail -3 gpurun_out/ncu_ws.log
