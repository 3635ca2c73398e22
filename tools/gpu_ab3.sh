# A/B of the systems kernels only: default, variants/*.so, default
echo default; timeout 300 python tools/ws_ab.py 2>&1 | tail -2
for v in variants/*.so; do echo $v; FC_LIB_PATH=$v timeout 300 python tools/ws_ab.py 2>&1 | tail -2; done
echo default; timeout 300 python tools/ws_ab.py 2>&1 | tail -2
