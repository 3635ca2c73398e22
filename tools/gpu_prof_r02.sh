# round-2 ncu evidence: one --set full capture per kernel (each after its command ran clean)
set -x
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_step_ws -s 3 -c 1 -o gpurun_out/r02_ws_c5 -f python bench.py --steps 2 --warmup 1 --no-variants --cpu-seconds 0 --no-e2e > /dev/null 2>&1; echo ws rc=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_step_ws -s 2 -c 1 -o gpurun_out/r02_ws_t3 -f python tools/prof_step.py --config C3 --level 8 --m 32 --steps 4 --skip 0 > /dev/null 2>&1; echo t3 rc=$?
