#!/bin/bash
# A/B timing of library builds under one env: tools/ab_lib.sh <config> <rounds> lib1 lib2 ...  ("" = in-tree)
C=$1; R=$2; shift 2
for i in $(seq $R); do
  for lib in "$@"; do
    KNB_LIB=$lib timeout 600 python bench.py --config $C --no-e2e --no-cpu --steps 40 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('${lib:-base}', '$C', 'ms %.4f'%l['ms_per_step'], 'kern %.4f'%l['roofline']['kernel_ms'], 'frac %.3f'%l['roofline']['frac'], 'mhz', l.get('clocks',{}).get('sm_mhz'), l.get('clocks',{}).get('reasons'))"
  done
done
