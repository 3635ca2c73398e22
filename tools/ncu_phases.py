"""Per-phase breakdown of the step kernel from an ncu report: SASS split at BAR.SYNC, with
predicated-on thread instructions, fp64 instructions and stall samples per segment."""
import csv
import subprocess
import sys


def main(rep, cells):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[1]
    ci = {h: i for i, h in enumerate(hdr)}

    def num(x):
        try:
            return float(x.replace(",", ""))
        except Exception:
            return 0.0
    segs, cur = [], {"fp": 0, "all": 0, "stall": 0, "n": 0, "lds": 0, "sts": 0}
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        src = r[ci["Source"]].strip()
        toks = src.split()
        op = toks[1] if toks and toks[0].startswith("@") and len(toks) > 1 else (toks[0] if toks else "")
        ti = num(r[ci["Predicated-On Thread Instructions Executed"]])
        cur["all"] += ti
        if op.startswith(("DFMA", "DMUL", "DADD")):
            cur["fp"] += ti
        if op.startswith("LDS"):
            cur["lds"] += ti
        if op.startswith("STS"):
            cur["sts"] += ti
        cur["stall"] += num(r[ci["Warp Stall Sampling (All Samples)"]])
        cur["n"] += 1
        if "BAR.SYNC" in src or "BAR.RED" in src:
            segs.append(cur)
            cur = {"fp": 0, "all": 0, "stall": 0, "n": 0, "lds": 0, "sts": 0}
    segs.append(cur)
    tot = sum(s["stall"] for s in segs) or 1
    T = {k: sum(s[k] for s in segs) for k in ("fp", "all", "lds", "sts")}
    print(f"total per cell: instr {T['all']/cells:.0f} fp64 {T['fp']/cells:.0f} lds {T['lds']/cells:.0f} sts {T['sts']/cells:.0f}")
    for k, s in enumerate(segs):
        if s["all"] == 0 and s["stall"] == 0:
            continue
        print(f"seg {k:2d}: sass {s['n']:5d} instr/cell {s['all']/cells:7.1f} fp64/cell {s['fp']/cells:7.1f} "
              f"lds {s['lds']/cells:6.1f} sts {s['sts']/cells:5.1f} stall {s['stall']/tot:6.1%}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]))
