"""Registers / spills per function from `nvcc -Xptxas -v` output: python scripts/ptxas_summary.py log [substr]"""
import re
import sys

txt = open(sys.argv[1]).read().split("\n")
sub = sys.argv[2] if len(sys.argv) > 2 else ""
cur = None
info = {}
for line in txt:
    m = re.search(r"Function properties for (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        info.setdefault(cur, {})["spill"] = f"st {m.group(1)} ld {m.group(2)}"
    m = re.search(r"Used (\d+) registers", line)
    if m:
        info.setdefault(cur, {})["regs"] = m.group(1)
for k, v in info.items():
    if sub in k:
        print(f"{k[-70:]:72s} regs={v.get('regs', '-'):>4s} spill={v.get('spill', '-')}")
