#!/bin/bash
# per-kernel device times (ncu, serialized, cold) for one sync step of each codec
GS=${1:-resnet50_161}; shift
for c in "$@"; do
  extra=""
  [ "$c" = "topk" ] && extra="--sparsity 0.99"
  [ "$c" = "randk" ] && extra="--sparsity 0.99"
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" -c 40 --csv --log-file gpurun_out/ll_$c.csv \
    python bench.py --codec $c --gradset $GS --steps 2 --warmup 1 --no-search --no-cpu-baseline --e2e-steps 1 $extra > /dev/null 2>&1
  echo "== $c"
  python - "$c" <<'PY'
import csv, sys, collections
rows = list(csv.reader(open(f"gpurun_out/ll_{sys.argv[1]}.csv")))
hdr = None; agg = collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID": hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r)); k = d["Kernel Name"].split("(")[0].replace("void mc::<unnamed>::", "")
        agg.setdefault(k, []).append(float(d["Metric Value"].replace(",","")))
# the e2e leg launches the fused kernels per 8 MB chunk: report the whole-group launches
# (>= half the longest) separately from the mean over all launches
for k, v in agg.items():
    big = [x for x in v if x >= 0.5 * max(v)]
    print(f"  {k[:60]:60s} n={len(v):3d} mean={sum(v)/len(v)/1000:8.1f} us"
          f"  whole-group n={len(big):3d} mean={sum(big)/len(big)/1000:8.1f} us")
PY
done
