"""Small runs through every kernel family, for compute-sanitizer (one tool per call):

    compute-sanitizer --tool memcheck  python tools/sanitize_cases.py
    compute-sanitizer --tool racecheck python tools/sanitize_cases.py
    compute-sanitizer --tool synccheck python tools/sanitize_cases.py

dense DMMA pass + finalize / reduce / geometry (c1 shape), kmeans++ device loop,
the twelve-warp MTI kernel (d = 32, k = 24), the eight-warp MTI kernel (d = 8),
the exact MTI walk, the tcgen05 f32 pass (CTA pairs, TMEM) with its rerank and
segmented sums, the tcgen05 MTI pass for f64 rows (d = 16) and its delta kernel,
and a semi-external run with the HBM row cache."""
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, ".")
import paper_1606_08905_b200 as kb  # noqa: E402
from paper_1606_08905_b200.outofcore import CacheSchedule, RowStore, kmeans_ondisk  # noqa: E402

S = kb.synth


def run(tag, m, **cfg):
    r = kb.kmeans(m, kb.EngineConfig(**cfg))
    print(f"{tag}: {r.n_iterations} iterations, counts {int(r.centroids.counts.sum())}", flush=True)


run("dense c1-shape", S.mixture(S.MixtureSpec(4000, 16, 8, 1, "uniform", -10, 10, 1.0)), k=8, pruning=False, max_iters=6)
run("kmeans++ + w12 MTI", S.mixture(S.MixtureSpec(6000, 32, 24, 2, "uniform", -5, 5, 1.0)), k=24, init="kmeanspp",
    seed=2, max_iters=6)
run("eight-warp MTI d8", S.mixture(S.MixtureSpec(6000, 8, 10, 3, "uniform", -1, 1, 0.1)), k=10, max_iters=6,
    mti_scan="dense")
run("exact MTI walk", S.mixture(S.MixtureSpec(3000, 8, 10, 3, "uniform", -1, 1, 0.1)), k=10, max_iters=5,
    mti_scan="exact")
run("tcgen05 f32 dense", S.mixture(S.MixtureSpec(1000, 64, 300, 5, "normal", 0, 0, 0.3, None, "float32")), k=300,
    pruning=False, max_iters=3)
run("tcgen05 MTI f64 d16", S.uniform(3000, 16, 4), k=100, max_iters=5, mti_scan="tc")
m = S.mixture(S.MixtureSpec(4000, 8, 6, 7, "uniform", -3, 3, 1.0))
with tempfile.TemporaryDirectory() as td:
    p = os.path.join(td, "m.knrm")
    kb.save_matrix(m, p)
    with RowStore.open(p) as store:
        r = kmeans_ondisk(store, kb.EngineConfig(k=6, seed=2, T=2, max_iters=8, mode="sem"),
                          cache_capacity=m.nbytes // 2, schedule=CacheSchedule(2))
print(f"semi-external: {r.n_iterations} iterations", flush=True)
print("sanitize cases done")
