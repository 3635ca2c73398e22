"""Instruction mix of an ncu report's SASS source page: warp-instructions executed per opcode
(and per cell-update when --cells is given), plus stall samples per opcode.
usage: ncu -i rep --page source --csv --print-source sass > x.csv; python tools/sass_mix.py x.csv [--cells N]"""
import csv
import sys
from collections import defaultdict


def main(path, cells=None):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    ex = defaultdict(float)
    th = defaultdict(float)
    st = defaultdict(float)
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        src = r[ix["Source"]].strip()
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        op = op.split(".")[0]
        ex[op] += float(r[ix["Instructions Executed"]] or 0)
        th[op] += float(r[ix["Predicated-On Thread Instructions Executed"]] or 0)
        st[op] += float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    tot = sum(ex.values())
    tst = sum(st.values())
    print(f"total warp-instr {tot:.4g}" + (f"  per cell-update {32 * tot / cells:.1f} thread-slots" if cells else ""))
    for op in sorted(ex, key=lambda o: -ex[o])[:40]:
        per = f" {32 * ex[op] / cells:8.1f}/cu" if cells else ""
        print(f"{op:10s} {ex[op]:14.4g} {100 * ex[op] / tot:6.2f}%{per}  active-lanes {th[op] / max(ex[op], 1):5.1f}  stall {100 * st[op] / max(tst, 1):5.1f}%")


if __name__ == "__main__":
    cells = None
    if "--cells" in sys.argv:
        cells = float(sys.argv[sys.argv.index("--cells") + 1])
    main(sys.argv[1], cells)
