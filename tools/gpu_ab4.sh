# A/B of the scalar sweeps (T1 / T2 / T4) on the default build and each variants/*.so; then the
# parity tests on the default
VARIANTS="default $(ls variants/*.so | xargs -n1 basename | sed 's/\.so$//')" ONLY=T1,T2,T4 bash tools/cv_variants.sh 2>&1 | grep -v "^$"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_ab4.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_ab4.log
