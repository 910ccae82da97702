"""Opcode mix of one kernel from `ncu -i X --page source --csv --print-source sass`:
executed warp instructions per opcode (and per element when --elems is given), plus the
stall-sample share.  Usage: python scripts/sass_mix.py file.csv [--elems N]"""
import csv
import sys
from collections import Counter

path = sys.argv[1]
elems = float(sys.argv[sys.argv.index("--elems") + 1]) if "--elems" in sys.argv else None
rows = list(csv.reader(open(path)))
hdr = rows[1]
ci, cs, ce = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
ops, stalls = Counter(), Counter()
tot = 0
for r in rows[2:]:
    if len(r) <= ce or not r[ce].isdigit():
        continue
    op = r[ci].strip().split()[0]
    if op.startswith("@"):
        op = r[ci].strip().split()[1]
    n = int(r[ce])
    ops[op] += n
    stalls[op] += int(r[cs] or 0)
    tot += n
ts = sum(stalls.values())
print(f"total warp instructions {tot}" + (f"  ({tot * 32 / elems:.1f} thread-instr / element)" if elems else ""))
for op, n in ops.most_common(40):
    extra = f"  {n * 32 / elems:6.2f}/elem" if elems else ""
    print(f"{op:28s} {n:12d} {100 * n / tot:5.1f}%{extra}  stall {100 * stalls[op] / max(ts, 1):5.1f}%")
