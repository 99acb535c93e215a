for i in 1 2; do for lib in variants/h5.so ""; do
for c in c3 c1; do
KNB_LIB=$lib timeout 600 python bench.py --config $c --no-e2e --no-cpu --steps 40 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('${lib:-base}', '$c', 'ms %.4f'%l['ms_per_step'], 'frac %.3f'%l['roofline']['frac'], 'k1 %.4f'%l['roofline_k1']['kernel_ms'], 'k1frac %.3f'%l['roofline_k1']['frac'])"
done
KNB_LIB=$lib timeout 900 python bench.py --config c4 --n 200000000 --no-e2e --no-cpu --steps 3 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('${lib:-base}', 'c4/200M', 'ms %.3f'%l['ms_per_step'], 'frac %.3f'%l['roofline']['frac'], 'k1frac %.3f'%l['roofline_k1']['frac'])"
done; done
