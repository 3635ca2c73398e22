"""Static SASS census of a step-kernel instantiation, split at barriers (BAR.SYNC / BAR.RED):
instructions, fp64 ops, spills and selects per phase.  Quick proxy between ncu runs.

    python tools/sass_phases.py EulerRoe 16 352 2
"""
import re
import subprocess
import sys
from collections import Counter

LIB = "paper_1308_1472_b200/libfc.so"


def main(solver, T, NT, MB):
    name = f"_ZN2fc6k_stepINS_{len(solver)}{solver}ELi{T}ELi{NT}ELi{MB}EEEvNS_8StepArgsEi"
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    start = out.find(f"Function : {name}")
    if start < 0:
        raise SystemExit(f"{name} not found")
    end = out.find("Function :", start + 10)
    body = out[start:end if end > 0 else None]
    segs = [Counter()]
    for line in body.splitlines():
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
        if not m:
            continue
        op = m.group(2)
        base = op.split(".")[0]
        segs[-1]["all"] += 1
        segs[-1][base] += 1
        if base.startswith("BAR"):
            segs.append(Counter())
    for k, c in enumerate(segs):
        fp = c["DFMA"] + c["DMUL"] + c["DADD"]
        print(f"seg {k:2d}: {c['all']:5d} instr, fp64 {fp:4d}, LDS {c['LDS']:3d} STS {c['STS']:3d} "
              f"STL {c['STL']:3d} LDL {c['LDL']:3d} IMAD {c['IMAD']:3d} FSEL/SEL {c['FSEL'] + c['SEL']:3d} "
              f"DSETP {c['DSETP']:3d} MUFU {c['MUFU']:2d}")
    tot = sum(segs, Counter())
    print("total", tot["all"], "fp64", tot["DFMA"] + tot["DMUL"] + tot["DADD"])


if __name__ == "__main__":
    main(*sys.argv[1:5])
