"""Full-size trajectory goldens for BASELINE configs c2 and c3, made by running the
REFERENCE package (numakmeans) on the exact bytes the GPU tests regenerate.

TEST INFRASTRUCTURE ONLY.  Run in the build container, where the reference is
mounted read-only (about 5 min for c2 and 20-30 min for c3 on 8 cores):

    PYTHONPATH=/root/reference/pkg/src:. python oracle/make_golden_full.py c2 c3

SURVEY.md section 8(c) prescribes full trajectories for C1-C3 (C1 is
``tests/golden/c1_full.npz``).  The reference's ``kmeans(matrix, EngineConfig(...))``
(engine.py:489-500) runs with the config's k / init / seed / pruning / tolerance /
max_iters, T = 8 threads (the merge is per task, engine.py:10-13, so T only moves
last-ulp rounding of the sums) and ``collect_assignments=True``.  Stored, compactly:

* ``history_sha``     sha256 of the int32 assignment vector after every iteration
                      (engine.py:408-409);
* ``sample_rows`` / ``sample_history``  the assignments of every STRIDE-th row after
                      every iteration (locates a mismatch without the whole history);
* ``assignments``     final assignments (uint8, k <= 255);
* every per-iteration counter (reassignments, dist_comps, skips, pruned_stale,
  pruned_tight), WCSS, the iteration count, ``converged``, the final centroid set
  and the reference's own initial centroids (centroids.py:131-189).

Nothing here travels to the GPU box: only the .npz outputs are committed.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_1606_08905_b200.synth import CONFIGS  # noqa: E402

OUT = os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "full")
STRIDE = 997


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int32).tobytes()).hexdigest()


def run(name: str, threads: int) -> None:
    from numakmeans import EngineConfig, init_centroids, kmeans  # the reference itself

    c = CONFIGS[name]
    t0 = time.perf_counter()
    m = c["data"](c["n"])
    t_gen = time.perf_counter() - t0
    cfg = EngineConfig(k=c["k"], init=c["init"], seed=int(name[1:]), pruning=c["pruning"],
                       max_iters=c["max_iters"], tolerance=c["tolerance"], T=threads,
                       collect_assignments=True)
    t0 = time.perf_counter()
    res = kmeans(m, cfg)
    dt = time.perf_counter() - t0
    init_c = init_centroids(m, cfg.k, cfg.init, cfg.seed, None)
    its = res.iterations
    rows = np.arange(0, m.shape[0], STRIDE, dtype=np.int64)
    hist = np.stack([h[rows] for h in res.assignment_history]).astype(np.uint8)
    os.makedirs(OUT, exist_ok=True)
    np.savez_compressed(
        os.path.join(OUT, f"{name}.npz"),
        n=np.array(m.shape[0]), d=np.array(m.shape[1]),
        means=res.centroids.means, prev_means=res.centroids.prev_means,
        counts=res.centroids.counts, drift=res.centroids.drift,
        assignments=res.assignments.astype(np.uint8),
        init_means=init_c.means,
        converged=np.array(res.converged),
        reassignments=np.array([s.reassignments for s in its], dtype=np.int64),
        wcss=np.array([s.wcss for s in its]),
        dist_comps=np.array([s.dist_comps for s in its], dtype=np.int64),
        skips=np.array([s.skips for s in its], dtype=np.int64),
        pruned_stale=np.array([s.pruned_stale for s in its], dtype=np.int64),
        pruned_tight=np.array([s.pruned_tight for s in its], dtype=np.int64),
        history_sha=np.array([sha(h) for h in res.assignment_history]),
        sample_rows=rows, sample_history=hist,
        data_sha=np.array(hashlib.sha256(m[:: max(1, m.shape[0] // 4096)].tobytes()).hexdigest()),
        threads=np.array(threads), ref_seconds=np.array(dt),
    )
    print(f"{name}: n={m.shape[0]} d={m.shape[1]} k={cfg.k} iters={res.n_iterations} "
          f"converged={res.converged} (data {t_gen:.1f}s, reference {dt:.1f}s, T={threads})", flush=True)


if __name__ == "__main__":
    th = int(os.environ.get("KNB_REF_THREADS", os.cpu_count() or 1))
    for nm in sys.argv[1:] or ["c2", "c3"]:
        run(nm, th)
