#!/bin/bash
# A/B of the dense pass (roofline_k1) between library builds: tools/ab_k1.sh <config> <rounds> lib...
C=$1; R=$2; shift 2
for i in $(seq $R); do
  for lib in "$@"; do
    KNB_LIB=$lib timeout 600 python bench.py --config $C --no-e2e --no-cpu --steps 40 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('${lib:-base}', '$C', 'ms %.4f'%l['ms_per_step'], 'k1 %.4f'%l['roofline_k1']['kernel_ms'], 'k1frac %.3f'%l['roofline_k1']['frac'])"
  done
done
