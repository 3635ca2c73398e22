# compute-sanitizer on small runs of the round-2 kernels (warp-sweep systems kernel, octree step)
cat > /tmp/san_ws.py <<'PY'
import sys; sys.path.insert(0, '.')
from paper_1308_1472_b200 import fc, fc3
from workloads.configs import c5, c3
from workloads.octree import forest3
import numpy as np
for w in (c5(level=1, m=16, steps=2), c3(level=0, m=32, steps=2)):
    fc.run(w, skip_quiescent=0)
f = forest3((2, 1, 1), 1)
fc3.run3(f, 8, np.random.default_rng(0).random((f.num_patches, 8, 8, 8)), (0.5, 0.3, -0.2), 0.01, 2)
print("ok")
PY
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python /tmp/san_ws.py > gpurun_out/san_$tool.log 2>&1; echo $tool rc=$?; tail -3 gpurun_out/san_$tool.log
done
