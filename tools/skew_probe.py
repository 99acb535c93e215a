"""§8(f) f4 probe: does the MTI pass balance when the active rows cluster in row ranges?

The same c2-law matrix is run in its generated order and with its rows sorted by
their initial cluster (so clause-1 survivors, which concentrate near cluster
boundaries, arrive in long contiguous runs).  The compacted MTI kernel deals
32-row blocks round-robin over all warps, so both orders should cost the same.
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1606_08905_b200 as kb  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = kb.synth.CONFIGS[name]
m = cfg["data"](cfg["n"])
first = kb.kmeans(m, kb.EngineConfig(k=cfg["k"], init="forgy", seed=int(name[1:]), pruning=True, max_iters=1))
# same starting centroids for both orders: the runs are identical up to the row permutation
ec = kb.EngineConfig(k=cfg["k"], init="given", initial_centroids=first.centroids.prev_means, pruning=True,
                     max_iters=40)
orders = {"generated": np.arange(m.shape[0]), "sorted by cluster": np.argsort(first.assignments, kind="stable")}
for label, order in orders.items():
    x = torch.from_numpy(np.ascontiguousarray(m[order])).cuda()
    r = kb.Lloyd(x, ec, ignore_stop=True)
    r.ctx.enqueue(6)
    torch.cuda.synchronize()
    K = 20
    t0 = time.perf_counter()
    r.ctx.enqueue(K)
    r.sync()
    el = (time.perf_counter() - t0) / K
    st = r.ctx.stats()[6:6 + K]
    print(f"{name} {label:>18}: {el * 1e3:.3f} ms/iter  skipped {np.mean([s.skips for s in st]) / m.shape[0]:.2f}",
          flush=True)
    r.close()
