"""Octree variant alone (bench.py's run_octree) with the kernel split from the library's timers."""
import argparse, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench
a = argparse.Namespace(warmup=3, variant_steps=20)
print(json.dumps(bench.run_octree(a, 6547.8)))
