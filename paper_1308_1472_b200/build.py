"""Build libfc.so in-tree with nvcc for sm_100a (no JIT, no torch extension machinery).

    python -m paper_1308_1472_b200.build [--force] [--verbose]

The library links the NCCL that ships with the torch wheel (so torch and libfc load one NCCL)
and the CUDA runtime statically.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libfc.so")
SOURCES = ["api.cu", "kernels.cu", "step.cu", "plan.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    cands = []
    if spec and spec.submodule_search_locations:
        for loc in spec.submodule_search_locations:
            cands.append(os.path.join(loc, "nccl"))
    for c in cands:
        if os.path.exists(os.path.join(c, "include", "nccl.h")):
            return os.path.join(c, "include"), os.path.join(c, "lib")
    raise RuntimeError("NCCL (nvidia-nccl wheel) not found")


def _deps():
    return [os.path.join(CSRC, s) for s in SOURCES] + glob.glob(os.path.join(CSRC, "*.h")) + \
        glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "fc.h"), __file__]


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    lib = out or LIB
    if not force and os.path.exists(lib):
        t = os.path.getmtime(lib)
        if all(os.path.getmtime(d) <= t for d in _deps()):
            return lib
    inc, libdir = nccl_dirs()
    tmp = lib + f".tmp{os.getpid()}"
    cmd = ["nvcc", *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-shared",
           "-cudart", "static", f"-I{inc}", f"-I{os.path.join(ROOT, 'include')}",
           "-Xptxas", "-v" if verbose else "-O3", *[f"-D{d}" for d in defines],
           "-o", tmp] + [os.path.join(CSRC, s) for s in SOURCES] + \
          [f"-L{libdir}", "-l:libnccl.so.2", "-Xlinker", f"-rpath,{libdir}"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libfc.so")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    # tuning builds: --define NAME=VALUE ... --out PATH (FC_LIB_PATH=PATH loads it)
    defs = [sys.argv[i + 1] for i, a in enumerate(sys.argv) if a == "--define"]
    outs = [sys.argv[i + 1] for i, a in enumerate(sys.argv) if a == "--out"]
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv, defines=defs,
                out=outs[0] if outs else None))
