"""CPU oracle for the semi-external I/O accounting of ``numakmeans`` (outofcore.py).

TEST INFRASTRUCTURE ONLY (see oracle/lloyd.py's header): the GPU path computes
these counters on the device (csrc/sem.cu); tests compare the two.

Given which rows each iteration fetches (``lloyd(..., collect_fetch=True)``),
restates, per iteration t:

* tasks: the T partition ranges split into task_size blocks
  (engine.py:215-220, scheduler.py:152-166); one fetch call per task -- every
  row of the task on a full pass (task_rows, outofcore.py:327-328), the task's
  clause-1 survivors on a pruned pass (rows_by_ids, :330-331; no call when none
  survive);
* fetch_rows (outofcore.py:163-225): bytes_requested += row_bytes per id;
  with a cache, hits / misses against the published index and only misses go
  to disk; bytes_read += page_size x total pages of page_runs over the misses
  (outofcore.py:118-145);
* the cache (RowCache, outofcore.py:228-270): rows_per_partition =
  (capacity // T) // row_bytes; at should_refresh(t) (outofcore.py:282-290)
  every id fetched during t is collected under its task's owner partition and,
  at the barrier, each partition keeps its smallest rows_per_partition ids; the
  published index is the union, used from iteration t + 1;
* rows_elided: the pruned pass's skips (note_elided, outofcore.py:334-337).

Pinned by tests/test_oracle_pins.py against tests/golden/sem/*.npz, made by
running the reference's ``kmeans_ondisk`` (oracle/make_golden_sem.py).
"""

from __future__ import annotations

import numpy as np

from oracle.lloyd import row_ranges


def should_refresh(t: int, start: int) -> bool:
    if t < start or t % start != 0:
        return False
    q = t // start + 1
    return q & (q - 1) == 0


def pages_of(ids: np.ndarray, row_bytes: int, page_size: int) -> int:
    """page_runs' total: the number of distinct pages the ascending rows touch."""
    if ids.size == 0:
        return 0
    first = ids * row_bytes // page_size
    last = (ids * row_bytes + row_bytes - 1) // page_size
    # pages of row i not already covered by row i-1 (rows ascend, intervals are ordered)
    prev_last = np.concatenate(([-1], last[:-1]))
    return int(np.sum(last - np.maximum(first, prev_last + 1) + 1))


def io_counters(fetched: list[np.ndarray], skips: list[int], n: int, d: int, T: int, task_size: int,
                page_size: int, cache_enabled: bool, capacity: int, start: int) -> np.ndarray:
    """(iterations, 5) int64: bytes_requested, bytes_read, cache_hits, cache_misses, rows_elided."""
    rb = 8 * d
    R = (capacity // T) // rb if cache_enabled else 0
    ranges = row_ranges(n, T)
    cached = np.zeros(n, dtype=bool)
    out = np.zeros((len(fetched), 5), dtype=np.int64)
    for t, f in enumerate(fetched):
        req = hits = misses = pages = 0
        for lo, hi in ranges:
            for a in range(lo, hi, task_size):
                b = min(a + task_size, hi)
                ids = a + np.flatnonzero(f[a:b])
                if ids.size == 0:
                    continue
                req += ids.size
                if cache_enabled:
                    c = cached[ids]
                    hits += int(c.sum())
                    misses += int((~c).sum())
                    ids = ids[~c]
                pages += pages_of(ids, rb, page_size)
        out[t] = (req * rb, pages * page_size, hits, misses, skips[t])
        if cache_enabled and should_refresh(t, start):
            cached[:] = False
            if R > 0:
                for lo, hi in ranges:
                    cached[lo + np.flatnonzero(f[lo:hi])[:R]] = True
    return out


def cached_ids(fetched: list[np.ndarray], n: int, d: int, T: int, capacity: int, start: int) -> np.ndarray:
    """The published cache after the last iteration (ascending ids)."""
    R = (capacity // T) // (8 * d)
    last = None
    for t, f in enumerate(fetched):
        if should_refresh(t, start):
            last = f
    if last is None or R == 0:
        return np.zeros(0, dtype=np.int64)
    return np.concatenate([lo + np.flatnonzero(last[lo:hi])[:R] for lo, hi in row_ranges(n, T)]).astype(np.int64)
