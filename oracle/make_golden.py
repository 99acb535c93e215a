"""Generate tests/golden/*.npz by running the REFERENCE package on every case.

TEST INFRASTRUCTURE ONLY.  Run in the build container, where the reference is
mounted read-only:

    PYTHONPATH=/root/reference/pkg/src:. python oracle/make_golden.py [case ...]

The reference's ``kmeans(matrix, EngineConfig(...))`` (engine.py:489-500) runs
with its defaults (T=1, task_size=8192) and ``collect_assignments=True``; the
fixture keeps the final centroid set, assignments, per-iteration statistics,
a sha256 per iteration of the assignment vector, and the reference's own
initial centroids (centroids.py:131-189).  Nothing here travels to the GPU box:
only the .npz outputs are committed.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from oracle.golden_cases import CASES, case_cfg, case_data  # noqa: E402

OUT = os.path.join(os.path.dirname(__file__), "..", "tests", "golden")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int32).tobytes()).hexdigest()


def main(names):
    from numakmeans import EngineConfig, init_centroids, kmeans  # the reference itself

    os.makedirs(OUT, exist_ok=True)
    for name in names:
        m = case_data(name)
        c = case_cfg(name)
        init = c.pop("init", "forgy")
        initial = c.pop("initial", None)
        cfg = EngineConfig(init=init, initial_centroids=initial, collect_assignments=True, **c)
        t0 = time.perf_counter()
        res = kmeans(m, cfg)
        dt = time.perf_counter() - t0
        init_c = init_centroids(m.astype(np.float64), cfg.k, init, cfg.seed, initial)
        its = res.iterations
        k = res.centroids.means.shape[0]
        np.savez_compressed(
            os.path.join(OUT, f"{name}.npz"),
            means=res.centroids.means, prev_means=res.centroids.prev_means,
            counts=res.centroids.counts, drift=res.centroids.drift,
            assignments=res.assignments.astype(np.int16 if k < 32768 else np.int32),
            init_means=init_c.means,
            converged=np.array(res.converged),
            reassignments=np.array([s.reassignments for s in its], dtype=np.int64),
            wcss=np.array([s.wcss for s in its]),
            dist_comps=np.array([s.dist_comps for s in its], dtype=np.int64),
            skips=np.array([s.skips for s in its], dtype=np.int64),
            pruned_stale=np.array([s.pruned_stale for s in its], dtype=np.int64),
            pruned_tight=np.array([s.pruned_tight for s in its], dtype=np.int64),
            history_sha=np.array([sha(h) for h in res.assignment_history]),
        )
        print(f"{name}: n={m.shape[0]} d={m.shape[1]} k={k} iters={res.n_iterations} "
              f"converged={res.converged} ({dt:.1f}s)", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or list(CASES))
