"""Host <-> HBM staging throughput (the e2e leg's upload): a pageable f64 array of
`gb` GB (d = 16) uploaded into a context, best of three; KNB_STAGE_WORKERS /
KNB_STAGE_CHUNK_MB select the pool shape.

    python tools/stage_bench.py [gb]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1606_08905_b200 import _native  # noqa: E402

gb = float(sys.argv[1]) if len(sys.argv) > 1 else 16.0
n = int(gb * 1e9 / 128)
host = np.empty((n, 16))
host[:] = 0.5  # touched: resident pages, like a user's array
ctx = _native.Context(0, n, n, 0, 16, 8, False, 2, 0.0, None)
_native.lib().knb_staging_reserve(0)
best = 1e9
for _ in range(3):
    t = time.perf_counter()
    ctx.upload(host)
    best = min(best, time.perf_counter() - t)
print(f"workers={os.environ.get('KNB_STAGE_WORKERS', 8)} chunk_mb={os.environ.get('KNB_STAGE_CHUNK_MB', 8)} "
      f"upload {host.nbytes / 1e9:.1f} GB: {best:.3f} s = {host.nbytes / best / 1e9:.1f} GB/s  (cpus {os.cpu_count()})",
      flush=True)
ctx.close()
