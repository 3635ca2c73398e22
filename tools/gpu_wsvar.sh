# C5 / T3 timing: default build and each variants/*.so
echo default; timeout 300 python tools/ws_ab.py 2>&1 | tail -2
for v in variants/*.so; do echo $v; FC_LIB_PATH=$v timeout 300 python tools/ws_ab.py --only C5 2>&1 | tail -1; done
echo default; timeout 300 python tools/ws_ab.py --only C5 2>&1 | tail -1
