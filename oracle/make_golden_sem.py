"""Generate tests/golden/sem/*.npz by running the REFERENCE's kmeans_ondisk.

TEST INFRASTRUCTURE ONLY.  Run in the build container, where the reference is
mounted read-only:

    PYTHONPATH=/root/reference/pkg/src:. python oracle/make_golden_sem.py [case ...]

Each case (oracle/golden_cases.py:SEM_CASES) writes its matrix as a raw file
under /tmp, runs ``kmeans_ondisk(RowStore(...), EngineConfig(mode="sem", ...),
...)`` (outofcore.py:440-455) with ``collect_assignments=True`` and keeps the
per-iteration IoDelta, skips, a sha256 per iteration of the assignment vector,
the final means and the published cache's row ids.
"""

from __future__ import annotations

import hashlib
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from oracle.golden_cases import SEM_CASES, sem_case  # noqa: E402

OUT = os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "sem")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int32).tobytes()).hexdigest()


def main(names):
    from numakmeans import outofcore
    from numakmeans.engine import EngineConfig

    os.makedirs(OUT, exist_ok=True)
    for name in names:
        m, cfg, io, page, start = sem_case(name)
        n, d = m.shape
        holder = {}

        class Spy(outofcore._DiskSource):
            def __init__(self, *a, **kw):
                super().__init__(*a, **kw)
                holder["src"] = self

        with tempfile.TemporaryDirectory() as tmp:
            path = os.path.join(tmp, "m.raw")
            m.astype("<f8").tofile(path)
            orig = outofcore._DiskSource
            outofcore._DiskSource = Spy
            try:
                with outofcore.RowStore(path, n, d, page_size=page) as store:
                    res = outofcore.kmeans_ondisk(store, EngineConfig(mode="sem", collect_assignments=True, **cfg),
                                                  schedule=outofcore.CacheSchedule(start), **io)
            finally:
                outofcore._DiskSource = orig
        cache = holder["src"].cache
        cached = np.array(sorted(cache.published), dtype=np.int64) if cache is not None else np.zeros(0, np.int64)
        its = res.iterations
        np.savez_compressed(
            os.path.join(OUT, f"{name}.npz"),
            io=np.array([[s.io.bytes_requested, s.io.bytes_read, s.io.cache_hits, s.io.cache_misses,
                          s.io.rows_elided] for s in its], dtype=np.int64),
            skips=np.array([s.skips for s in its], dtype=np.int64),
            reassignments=np.array([s.reassignments for s in its], dtype=np.int64),
            history_sha=np.array([sha(h) for h in res.assignment_history]),
            means=res.centroids.means,
            cached_ids=cached,
            converged=np.array(res.converged),
        )
        tot = res.io_totals
        print(f"{name}: n={n} d={d} iters={res.n_iterations} req={tot.bytes_requested} read={tot.bytes_read} "
              f"hits={tot.cache_hits} misses={tot.cache_misses} cached={cached.size}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or list(SEM_CASES))
