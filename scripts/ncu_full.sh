#!/bin/bash
# ncu --set full of every kernel of one sync step per codec (N=1, merged partition, R50 set).
# Reports land in gpurun_out/full_<codec>.ncu-rep; read them here with `ncu -i`.
GS=${GS:-resnet50_161}
COUNT=${COUNT:-8}
for c in "$@"; do
  extra=""
  [ "$c" = "topk" ] && extra="--sparsity 0.99"
  [ "$c" = "randk" ] && extra="--sparsity 0.99"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^k_" -c $COUNT -f -o gpurun_out/full_$c \
    python bench.py --codec $c --gradset $GS --steps 1 --warmup 1 --no-search --no-cpu-baseline --e2e-steps 1 $extra \
    > gpurun_out/full_$c.log 2>&1
  echo "$c rc=$?"
done
