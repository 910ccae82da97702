#!/bin/bash
# one bench line per codec on a gradient set (N=1, merged partition, no CPU baseline)
GS=${1:-resnet50_161}
shift
MODE="$*"  # extra bench args (e.g. --graph / --eager)
for c in efsignsgd onebit int8 qsgd terngrad dgc_lite topk randk threshold signsgd signum fp16 identity; do
  extra=""
  [ "$c" = "topk" ] && extra="--sparsity 0.99"
  [ "$c" = "randk" ] && extra="--sparsity 0.99"
  timeout 300 python bench.py --codec $c --gradset $GS --steps 50 --warmup 5 --no-search --no-cpu-baseline --e2e-steps 3 $extra $MODE 2>&1 | tail -1 | python -c "
import json,sys
try:
    d=json.loads(sys.stdin.read())
    print('$c', round(d['value'],1), 'GB/s  step_ms', round(d['ms_per_step'],4), ' kern_ms', d['roofline']['kernel_ms'], ' launches/step', d['gpu_launches']/d['steps'])
except Exception as e:
    print('$c', 'FAILED', e)
"
done
