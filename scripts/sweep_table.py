"""Render the measured sweeps under profiles/ as DESIGN.md's table rows.

    python scripts/sweep_table.py profiles/r1_codec_sweep.txt
    python scripts/sweep_table.py partition profiles/r1_partition_sweep_vgg16.jsonl
    python scripts/sweep_table.py projection profiles/r1_projection_multi_gpu.jsonl
"""

import re
import sys

SETS = ["resnet50_161", "resnet101_314", "maskrcnn_201", "vgg16_32"]


def parse(path):
    out, cur = {}, None
    for line in open(path):
        if line.startswith("## "):
            cur = line[3:].strip()
            out[cur] = {}
            continue
        m = re.match(r"(\w+) ([\d.]+) GB/s", line)
        if m and cur:
            out[cur][m.group(1)] = float(m.group(2))
    return out


def codec_rows(path):
    res = parse(path)
    codecs = list(res[SETS[0]])
    for c in codecs:
        cells = [f"{res[s].get(c, float('nan')):.0f}" for s in SETS if s in res]
        cells[0] = f"**{cells[0]}**"
        print(f"| {c} | " + " | ".join(cells) + " |")


def partition_rows(path):
    """Rows of DESIGN.md's partition-count tables from scripts/partition_sweep.py output."""
    import json
    rows = {}
    for line in open(path):
        r = json.loads(line)
        d = rows.setdefault(r["codec"], {"naive": {}, "analytic_opt": {}, "heuristic_search": None})
        if r["partition"] == "heuristic_search":
            d["heuristic_search"] = r
        else:
            d[r["partition"]][r["y"]] = r["GBps"]
    for c, d in rows.items():
        naive = " | ".join(f"{d['naive'][y]:.0f}" if y in d["naive"] else "" for y in range(1, 9))
        ana = " / ".join(f"{d['analytic_opt'][y]:.0f}" for y in (2, 3) if y in d["analytic_opt"])
        h = d["heuristic_search"]
        hs = f"{h['GBps']:.0f} (y={len(h['boundaries']) + 1})" if h else ""
        print(f"| {c} | {naive} | {ana} | {hs} |")


def projection_rows(path):
    import json
    rows = {}
    for line in open(path):
        r = json.loads(line)
        rows.setdefault(r["codec"], {})[r["N"]] = r
    for c, d in rows.items():
        cells = [f"{d[1]['per_gpu_GBps']:.0f}"]
        cells += [f"{d[n]['per_gpu_GBps']:.0f} / {d[n]['p2p_per_gpu_GBps']:.0f}" for n in (2, 4, 8) if n in d]
        print(f"| {c} | " + " | ".join(cells) + " |")


if __name__ == "__main__":
    kind, path = (sys.argv[1], sys.argv[2]) if len(sys.argv) > 2 else ("codecs", sys.argv[1])
    {"codecs": codec_rows, "partition": partition_rows, "projection": projection_rows}[kind](path)
