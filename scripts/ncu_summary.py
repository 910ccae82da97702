"""Summarise `ncu --page details --csv` output: one block per kernel launch with the
speed-of-light, issue, occupancy and pipe numbers used in DESIGN.md.

    python scripts/ncu_summary.py details.csv [raw.csv]
"""
import csv
import sys

KEEP = ("Duration", "DRAM Throughput", "Compute (SM) Throughput", "Issue Slots Busy", "Executed Ipc Active",
        "Registers Per Thread", "Achieved Occupancy", "Eligible Warps Per Scheduler", "Grid Size", "Block Size")
RAW = ("sm__pipe_fmaheavy_cycles_active.sum.pct_of_peak_sustained_elapsed",
       "sm__inst_executed_pipe_alu.sum.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_xu.sum.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
       "dram__bytes_read.sum", "dram__bytes_write.sum")


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    h = rows[0]
    ki, mi, vi, ui, ii = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    out = {}
    for r in rows[1:]:
        if r[mi] in KEEP:
            out.setdefault((r[ii], r[ki]), []).append(f"{r[mi]} = {r[vi]} {r[ui]}".rstrip())
    raw = {}
    if len(sys.argv) > 2:
        rr = list(csv.reader(open(sys.argv[2])))
        hh = rr[0]
        for r in rr[2:]:
            raw[r[hh.index("ID")]] = [f"{k} = {r[hh.index(k)]}" for k in RAW if k in hh]
    for (i, k), v in out.items():
        print(f"[{i}] {k[:110]}")
        for x in v + raw.get(i, []):
            print("    " + x)


if __name__ == "__main__":
    main()
