# variant timing (T1-T4 + O3): default build and variants/*.so
echo default; timeout 600 python tools/var_ab.py 2>&1 | grep '^{' | head -4
for v in variants/*.so; do echo $v; FC_LIB_PATH=$v timeout 600 python tools/var_ab.py 2>&1 | grep '^{' | head -4; done
