# ncu captures of the scalar register-sweep kernels (T2: C2 physics L8 m16; T1: C1 physics L10 m8; T4: C4 physics L7/L8)
for cfg in "C2 8 16" "C1 10 8"; do set -- $cfg
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_step_cv -s 2 -c 1 -o gpurun_out/prof_cv_$1 -f python tools/prof_step.py --config $1 --level $2 --m $3 --steps 4 --skip 0 > gpurun_out/ncu_cv_$1.log 2>&1; echo ncu $1 rc=$?; done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_step_cvc -s 2 -c 1 -o gpurun_out/prof_cvc_C4 -f python tools/prof_step.py --config C4 --level 6 --steps 4 --skip 0 > gpurun_out/ncu_cvc.log 2>&1; echo ncu C4 rc=$?
