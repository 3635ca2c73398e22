# quick GPU check: the given pytest selection
timeout 1200 python -m pytest "$@" -x -q > gpurun_out/pytest_quick.log 2>&1; echo pytest rc=$?; tail -8 gpurun_out/pytest_quick.log
