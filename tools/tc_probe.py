"""Quick probe of the f32 tensor-core path on a small case (debug aid)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1606_08905_b200 as kb  # noqa: E402
from oracle import lloyd as O  # noqa: E402

n, d, k = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (2000, 64, 40)))
m = kb.synth.mixture(kb.synth.MixtureSpec(n, d, max(1, k // 2), 7, "normal", 0, 0, 0.3, None, "float32"))
cfg = kb.EngineConfig(k=k, init="forgy", seed=1, pruning=False, max_iters=4, collect_assignments=True)
s = kb.Lloyd(m, cfg)
print("describe", s.ctx.describe(), flush=True)
s.step()
s.sync()
print("tc_info after 1 step", s.ctx.tc_info(), flush=True)
a1 = s.ctx.assignments()
s.close()
o = O.lloyd(m.astype(np.float64), k, init="forgy", seed=1, pruning=False, max_iters=4, collect=True)
print("iter0 mismatches", int(np.sum(a1 != o.history[0])), flush=True)
t0 = time.time()
r = kb.kmeans(m, cfg)
print("kmeans", time.time() - t0, "iters", r.n_iterations, "oracle", o.n_iterations, flush=True)
for t, (a, b) in enumerate(zip(r.assignment_history, o.history)):
    print("iter", t, "mismatch", int(np.sum(a != b)))
print("means err", float(np.abs(r.centroids.means - o.means).max()))
print("wcss", [s.wcss for s in r.iterations], [s.wcss for s in o.iterations])
