"""Semi-external k-means: rows beyond HBM (numakmeans outofcore.py, section 8(f) f2).

The reference keeps the rows on disk, reads them at page granularity with a
partitioned row cache refreshed on an exponential schedule, and never reads the
rows that clause 1 of MTI skips (``kmeans_ondisk``, outofcore.py:440-455).  On a
B200 the tiers shift by one: HBM is the scarce "memory", host memory the "disk".

    RowStore            a KNRM or raw f64 matrix file, memory-mapped
    kmeans_ondisk       copies the payload once into host memory that the GPU maps
                        (knb_attach_host_rows) and runs the GPU engine with the rows
                        left there: every pass reads them over the host link, pruned
                        passes fetch only the survivors of clause 1, and an HBM row
                        cache with the reference's policy (T partitions, smallest ids
                        first, rebuilt at start, 3 start, 7 start, ...; csrc/sem.cu)
                        serves cached survivors from HBM
    IterationStats.io   the reference's I/O counters for the same run -- bytes
                        requested, page-granular bytes read, cache hits / misses,
                        rows elided -- computed exactly on the device

Limit: the payload must fit in host memory (kmeans_ondisk checks and raises
MemoryError); the reference streams pages from disk on demand instead.
Results (assignments, centroids, every per-iteration counter) equal the
in-memory engine's, as in the reference (test_sem.py).
"""

from __future__ import annotations

import dataclasses
import os
from dataclasses import dataclass

import numpy as np

from .fileio import HEADER_SIZE, read_header
from .matrix import MatrixFormatError

DEFAULT_PAGE_SIZE = 4096
DEFAULT_CACHE_BYTES = 64 * 1024 * 1024
DEFAULT_REFRESH_START = 5


class RowStore:
    """A row-major f64 matrix file: shape, page size (the unit of the I/O accounting)
    and a read-only memory map of the payload."""

    def __init__(self, path, n: int, d: int, page_size: int = DEFAULT_PAGE_SIZE, payload_offset: int = 0):
        if min(n, d) < 1:
            raise ValueError("n and d must be >= 1")
        if page_size < 1:
            raise ValueError("page_size must be >= 1")
        size = os.path.getsize(path)
        need = payload_offset + 8 * n * d
        if size != need:
            raise MatrixFormatError(f"{path}: {size} bytes on disk, expected {need} for {n} x {d} f64 rows")
        self.path, self.n, self.d = str(path), int(n), int(d)
        self.page_size, self.row_bytes = int(page_size), 8 * int(d)
        self.rows = np.memmap(self.path, dtype="<f8", mode="r", offset=payload_offset, shape=(self.n, self.d))

    @classmethod
    def open(cls, path, raw: bool = False, n: int | None = None, d: int | None = None,
             page_size: int = DEFAULT_PAGE_SIZE) -> "RowStore":
        """A KNRM file (shape from its header) or, with raw=True, a bare payload of n x d."""
        if not raw:
            hn, hd = read_header(path)
            return cls(path, hn, hd, page_size, HEADER_SIZE)
        if n is None or d is None:
            raise MatrixFormatError("raw files carry no shape; pass n and d explicitly")
        return cls(path, n, d, page_size)

    def read_all_into(self, out: np.ndarray, chunk_rows: int = 1 << 20) -> None:
        """The payload into ``out`` (n x d f64) in blocks of rows."""
        for a in range(0, self.n, chunk_rows):
            out[a:a + chunk_rows] = self.rows[a:a + chunk_rows]

    def close(self) -> None:
        mm = getattr(self.rows, "_mmap", None)
        self.rows = None
        if mm is not None:
            mm.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


@dataclass(frozen=True)
class CacheSchedule:
    """The HBM row cache is rebuilt at iteration ``start`` and then at doubling gaps:
    start, 3 start, 7 start, ... (the reference's schedule, outofcore.py:273-290)."""

    start: int = DEFAULT_REFRESH_START

    def __post_init__(self):
        if self.start < 1:
            raise ValueError("refresh start must be >= 1")


def _available_host_bytes() -> int | None:
    try:
        return os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
    except (ValueError, OSError, AttributeError):  # pragma: no cover - non-POSIX
        return None


def kmeans_ondisk(store: RowStore, cfg, *, cache_enabled: bool = True,
                  cache_capacity: int = DEFAULT_CACHE_BYTES,
                  schedule: CacheSchedule | None = None, inspect_cache: bool = False):
    """Cluster a file-resident matrix with the rows outside HBM (outofcore.py:440-455).

    Same results as ``kmeans()`` on the same matrix; ``IterationStats.io`` and
    ``KmeansResult.io_totals`` carry the reference's I/O accounting for this run;
    ``inspect_cache`` returns the final HBM cache as ``KmeansResult.row_cache``
    (ids, rows).  The payload is copied into host memory first: MemoryError when it
    does not fit.
    """
    from .engine import _run_sem
    if cfg.mode != "sem":
        raise ValueError("kmeans_ondisk() runs in sem mode; set cfg.mode='sem'")
    cfg.validate()
    if cache_capacity < 0:
        raise ValueError("cache capacity must be >= 0")
    need = store.n * store.row_bytes
    avail = _available_host_bytes()
    if avail is not None and need > avail:
        raise MemoryError(f"kmeans_ondisk: the {need} B payload does not fit the {avail} B of free host memory "
                          "(rows are staged in host memory, not streamed from disk)")
    sched = schedule or CacheSchedule()
    rows = np.empty((store.n, store.d), dtype=np.float64)  # anonymous: the driver can page-lock it
    store.read_all_into(rows)
    run_cfg = dataclasses.replace(cfg, host_rows=True)
    return _run_sem(rows, run_cfg, dict(T=cfg.T, task_size=cfg.task_size, page_size=store.page_size,
                                        cache_enabled=bool(cache_enabled), cache_capacity=int(cache_capacity),
                                        refresh_start=sched.start, inspect_cache=inspect_cache))
