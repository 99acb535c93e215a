#!/bin/bash
# A/B timing of an environment switch: tools/ab_env.sh VAR "<values>" <config> [rounds]
V=$1; VALS=$2; C=${3:-c2}; R=${4:-2}
for i in $(seq $R); do
  for val in $VALS; do
    env $V=$val timeout 600 python bench.py --config $C --no-e2e --no-cpu --steps 40 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$V=$val', '$C', 'ms %.4f'%l['ms_per_step'], 'kern %.4f'%l['roofline']['kernel_ms'], 'frac %.3f'%l['roofline']['frac'])"
  done
done
