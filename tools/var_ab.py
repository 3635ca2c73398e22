"""bench.py's T1-T4 + O3 variants alone (full update, CUDA events), one summary line each:
    [FC_REGULAR_RING=0] [FC_LIB_PATH=...] python tools/var_ab.py [--variant-steps 20]"""
import argparse, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench
from paper_1308_1472_b200 import fc
ap = argparse.ArgumentParser()
ap.add_argument("--variant-steps", type=int, default=20)
ap.add_argument("--warmup", type=int, default=3)
a = ap.parse_args()
out = bench.run_variants(a, fc, 6547.8)
for k, v in out.items():
    print(json.dumps({"v": k, "ms": round(v["ms_per_step"], 4), "G_per_s": round(v["value"] / 1e9, 2),
                      "hbm_frac": round(v["hbm_roofline_frac"], 3),
                      "graph_ms": round(v["graph"]["ms_per_step"], 4) if v.get("graph") else None,
                      "graph_frac": round(v["graph"]["hbm_roofline_frac"], 3) if v.get("graph") else None,
                      "regular": os.environ.get("FC_REGULAR_RING", "1")}))
