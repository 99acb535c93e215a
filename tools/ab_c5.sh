#!/bin/bash
# c5 A/B: step time, assign-pass time and the certificate counters per library build
for lib in "$@"; do
  KNB_LIB=$lib timeout 900 python bench.py --config c5 --no-e2e --no-cpu --steps 10 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$lib', 'ms %.3f'%l['ms_per_step'], 'kern %.3f'%l['roofline']['kernel_ms'], 'cert', l.get('tc_certificate'))"
done
