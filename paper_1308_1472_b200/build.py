"""Build libfc.so in-tree with nvcc for sm_100a (no JIT, no torch extension machinery).

    python -m paper_1308_1472_b200.build [--force] [--verbose]

The library links the NCCL that ships with the torch wheel (so torch and libfc load one NCCL)
and the CUDA runtime statically.
"""
from __future__ import annotations

import glob
import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libfc.so")
SOURCES = ["api.cu", "kernels.cu", "step.cu", "step_ws.cu", "step3.cu", "plan.cpp"]
# per-source extra flags: the octree path is bitwise the oracle (no fused multiply-add contraction)
EXTRA = {"step3.cu": ["-fmad=false"]}
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
        glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(CSRC, "plan3.cpp")] + \
        glob.glob(os.path.join(ROOT, "include", "*.h")) + [__file__]


def _stamp(cmd) -> str:
    """Content hash of every source, header and the exact nvcc command (defines, flags): the
    cache key of a built library.  A library whose stamp differs is rebuilt, whatever its mtime
    (a prebuilt .so shipped to another box is never trusted on its timestamp)."""
    h = hashlib.sha256()
    for d in sorted(_deps()):
        h.update(os.path.basename(d).encode())
        with open(d, "rb") as f:
            h.update(f.read())
    h.update("\0".join(cmd).encode())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    lib = out or LIB
    inc, libdir = nccl_dirs()
    tmp = lib + ".tmp"
    cmd = ["nvcc", *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-shared",
           "-cudart", "static", f"-I{inc}", f"-I{os.path.join(ROOT, 'include')}",
           "-Xptxas", "-O3", *[f"-D{d}" for d in defines],
           "-o", tmp] + [os.path.join(CSRC, s) for s in SOURCES] + \
          [f"-L{libdir}", "-l:libnccl.so.2", "-Xlinker", f"-rpath,{libdir}"]
    stamp = _stamp([os.path.relpath(c, ROOT) if c.startswith(ROOT) else c for c in cmd])
    stamp_file = lib + ".stamp"
    if not force and os.path.exists(lib) and os.path.exists(stamp_file):
        with open(stamp_file) as f:
            if f.read().strip() == stamp:
                return lib
    if verbose:
        cmd[cmd.index("-O3", cmd.index("-Xptxas"))] = "-v"
    # compile the translation units in parallel (step.cu dominates), then link
    odir = os.path.join(os.path.dirname(lib), "build", f"obj{os.getpid()}")
    os.makedirs(odir, exist_ok=True)
    pre = cmd[:cmd.index("-shared")] + cmd[cmd.index("-shared") + 1:cmd.index("-o")]
    procs, objs = [], []
    for s in SOURCES:
        o = os.path.join(odir, s + ".o")
        objs.append(o)
        procs.append((s, subprocess.Popen(pre + EXTRA.get(s, []) + ["-c", "-o", o, os.path.join(CSRC, s)],
                                          stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    failed = False
    for s, p in procs:
        out, err = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(out + err)
            failed = True
        elif verbose:
            sys.stderr.write(err)
    if failed:
        raise RuntimeError("nvcc failed building libfc.so")
    tmp = lib + f".tmp{os.getpid()}"
    link = ["nvcc", *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs,
            f"-L{libdir}", "-l:libnccl.so.2", "-Xlinker", f"-rpath,{libdir}"]
    res = subprocess.run(link, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed linking libfc.so")
    for o in objs:
        os.remove(o)
    os.rmdir(odir)
    os.replace(tmp, lib)
    with open(stamp_file, "w") as f:
        f.write(stamp + "\n")
    return lib


if __name__ == "__main__":
    # tuning builds: --define NAME=VALUE ... --out PATH (FC_LIB_PATH=PATH loads it)
    defs = [sys.argv[i + 1] for i, a in enumerate(sys.argv) if a == "--define"]
    outs = [sys.argv[i + 1] for i, a in enumerate(sys.argv) if a == "--out"]
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv, defines=defs,
                out=outs[0] if outs else None))
