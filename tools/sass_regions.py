"""Warp-instructions executed per source region of a kernel (ncu --page source --csv
--print-source cuda,sass dump): regions are (file, first line, last line, name) ranges given on
the command line as file:a-b=name; the rest is reported per file."""
import csv
import sys
from collections import defaultdict


def main(path, specs, cells=None):
    regs = []
    for s in specs:
        loc, name = s.split("=")
        f, ab = loc.split(":")
        a, b = ab.split("-")
        regs.append((f, int(a), int(b), name))
    rows = list(csv.reader(open(path)))
    f = None
    cur = None
    tot = defaultdict(float)
    fp = defaultdict(float)
    for r in rows:
        if r and r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if len(r) > 8 and r[0].isdigit():
            ln = int(r[0])
            cur = next((n for (ff, a, b, n) in regs if ff == f and a <= ln <= b), f)
            continue
        if len(r) > 8 and r[0] == "" and r[2].startswith("0x"):
            op = r[3].strip().split()
            if not op:
                continue
            o = (op[1] if op[0].startswith("@") else op[0]).split(".")[0]
            try:
                ex = float(r[7])
            except ValueError:
                continue
            tot[cur] += ex
            if o in ("DFMA", "DMUL", "DADD", "DSETP", "DMNMX"):
                fp[cur] += ex
    T = sum(tot.values())
    for k in sorted(tot, key=lambda k: -tot[k]):
        per = f"  {32 * tot[k] / cells:7.1f} /cu (fp64 {32 * fp[k] / cells:6.1f})" if cells else ""
        print(f"{k:24s} {100 * tot[k] / T:6.2f}%  fp64 {100 * fp[k] / max(tot[k], 1):5.1f}%{per}")


if __name__ == "__main__":
    args = [a for a in sys.argv[2:] if "=" in a]
    cells = float(sys.argv[sys.argv.index("--cells") + 1]) if "--cells" in sys.argv else None
    main(sys.argv[1], args, cells)
