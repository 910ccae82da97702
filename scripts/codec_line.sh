#!/bin/bash
# one compact bench line: codec gradset [extra bench args...]
c=$1; gs=$2; shift 2
timeout 300 python bench.py --codec $c --gradset $gs --steps 50 --warmup 5 --no-search --no-cpu-baseline --e2e-steps 3 "$@" 2>&1 | tail -1 | python -c "
import json,sys
try:
    d=json.loads(sys.stdin.read())
    print('$c $gs', round(d['value'],1), 'GB/s  step_ms', round(d['ms_per_step'],4), ' kern_ms', round(d['roofline']['kernel_ms'],4), ' launches/step', d['gpu_launches']/d['steps'])
except Exception as e:
    print('$c $gs FAILED', e)
"
