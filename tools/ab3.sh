#!/bin/bash
# A/B/C timing of library builds: tools/ab3.sh <config> <rounds> <lib>...
C=$1; R=$2; shift 2
for i in $(seq $R); do
  for lib in "$@"; do
    KNB_LIB=$lib timeout 600 python bench.py --config $C --no-e2e --no-cpu --steps 40 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$lib', '$C', 'ms %.4f'%l['ms_per_step'], 'kern %.4f'%l['roofline']['kernel_ms'], 'k1 %.4f'%(l.get('roofline_k1') or {}).get('kernel_ms', 0))"
  done
done
