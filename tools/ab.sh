#!/bin/bash
# A/B timing of two library builds: tools/ab.sh <variant.so> <config> [rounds]
V=$1; C=${2:-c2}; R=${3:-3}
for i in $(seq $R); do
  for lib in "" "$V"; do
    KNB_LIB=$lib timeout 600 python bench.py --config $C --no-e2e --no-cpu --steps 40 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('${lib:-base}', '$C', 'ms %.4f'%l['ms_per_step'], 'kern %.4f'%l['roofline']['kernel_ms'])"
  done
done
