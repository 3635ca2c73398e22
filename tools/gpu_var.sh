# variant timing: default build and variants/*.so (T1-T4 + O3), twice each
for r in 1 2; do
echo default; timeout 600 python tools/var_ab.py 2>&1 | grep '^{'
for v in variants/*.so; do echo $v; FC_LIB_PATH=$v timeout 600 python tools/var_ab.py 2>&1 | grep '^{'; done
done
