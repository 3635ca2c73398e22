# ncu --set full capture of the scalar register sweep on T1 (m = 8) and T2 (m = 16), source views exported
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_step_cv -s 2 -c 1 -o gpurun_out/prof_t1 -f python tools/prof_step.py --config C1 --level 10 --m 8 --steps 4 --skip 0 > /dev/null 2>&1; echo t1 rc=$?
ncu -i gpurun_out/prof_t1.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof_t1_src.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/prof_t1.ncu-rep 67108864
rm -f gpurun_out/prof_t1.ncu-rep
