"""Summarise an ncu --set full report (raw page) for the step kernel: time, occupancy, pipes,
fp64 instruction mix per cell-update, DRAM bytes, stall reasons."""
import csv
import subprocess
import sys


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    return [dict(zip(hdr, r)) for r in rows[2:]], dict(zip(hdr, units))


def f(v):
    try:
        return float(v.replace(",", ""))
    except Exception:
        return float("nan")


def main(rep, cells=None):
    rows, units = load(rep)
    for r in rows:
        name = r.get("Kernel Name", "")[:70]
        t = f(r["gpu__time_duration.sum"])
        tu = units["gpu__time_duration.sum"]
        t_s = t * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}.get(tu, 1e-9)
        cyc = f(r["smsp__cycles_active.avg"])
        el = f(r.get("sm__cycles_elapsed.avg", "nan"))
        fp = {k: f(r.get(f"smsp__sass_thread_inst_executed_op_{k}_pred_on.sum.per_cycle_elapsed", "nan"))
              for k in ("dfma", "dmul", "dadd")}
        print(f"kernel {name}")
        print(f"  time {t} {tu}; regs {r.get('launch__registers_per_thread')}; block {r.get('launch__block_size')}; "
              f"grid {r.get('launch__grid_size')}")
        print(f"  occupancy achieved {r.get('sm__warps_active.avg.pct_of_peak_sustained_active')} %; "
              f"fp64 pipe {r.get('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active')} % of active; "
              f"issue active {r.get('sm__inst_issued.avg.pct_of_peak_sustained_active')} %")
        dr = f(r["dram__bytes_read.sum"]) * (1e6 if units["dram__bytes_read.sum"] == "Mbyte" else (1e9 if units["dram__bytes_read.sum"] == "Gbyte" else 1))
        dw = f(r["dram__bytes_write.sum"]) * (1e6 if units["dram__bytes_write.sum"] == "Mbyte" else (1e9 if units["dram__bytes_write.sum"] == "Gbyte" else 1))
        print(f"  dram read {dr/1e6:.1f} MB write {dw/1e6:.1f} MB -> {(dr+dw)/t_s/1e9:.1f} GB/s")
        if cells:
            tot_fp = sum(fp.values()) * el if el == el else float("nan")
            print(f"  per cell-update: dram {(dr+dw)/cells:.1f} B; fp64 thread-instr {tot_fp/cells:.0f} "
                  f"(dfma {fp['dfma']*el/cells:.0f} dmul {fp['dmul']*el/cells:.0f} dadd {fp['dadd']*el/cells:.0f})")
        st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): f(v) for k, v in r.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
        tot = sum(v for v in st.values() if v == v)
        top = sorted(st.items(), key=lambda kv: -kv[1])[:8]
        print("  stalls: " + ", ".join(f"{k} {v/tot:.0%}" for k, v in top))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else None)
