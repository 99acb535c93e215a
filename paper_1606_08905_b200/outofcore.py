"""Semi-external k-means: rows beyond HBM (numakmeans outofcore.py, §8(f) f2).

The reference keeps the rows on disk, reads them at page granularity with a
partitioned row cache refreshed on an exponential schedule, and never reads the
rows clause 1 of MTI skips (``kmeans_ondisk``, outofcore.py:440-455).  On a B200
the tiers shift by one: HBM is the scarce "memory", host memory is the "disk".

    RowStore            the matrix file, read with positional I/O (host side)
    kmeans_ondisk       reads the payload once into page-locked host memory and
                        runs the GPU engine with the rows left there: every pass
                        reads them over the host link, pruned passes fetch only the
                        survivors of clause 1, and an HBM row cache (the
                        reference's RowCache policy, rebuilt on the device at the
                        should_refresh iterations) serves cached survivors from HBM
    IterationStats.io   the reference's I/O counters for the same run -- bytes
                        requested, page-granular bytes read, cache hits / misses,
                        rows elided -- computed exactly on the device

Results (assignments, centroids, every per-iteration counter) equal the
in-memory engine's, as in the reference (test_sem.py).  ``fetch_rows`` and
``page_runs`` are the reference's host-side helpers for reading rows from a
``RowStore`` (used by tools and tests; the GPU path never calls them).
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
    """Raw on-disk row-major f64 matrix read through positional I/O (outofcore.py:35-103).

    ``payload_offset`` lets a header-carrying file be streamed; page arithmetic is
    relative to the payload."""

    def __init__(self, path, n: int, d: int, page_size: int = DEFAULT_PAGE_SIZE, payload_offset: int = 0):
        if n < 1 or d < 1:
            raise ValueError("n and d must be >= 1")
        if page_size < 1:
            raise ValueError("page_size must be >= 1")
        self.path = str(path)
        self.n, self.d = int(n), int(d)
        self.page_size = int(page_size)
        self.payload_offset = int(payload_offset)
        self.row_bytes = 8 * self.d
        expected = self.payload_offset + self.n * self.d * 8
        actual = os.path.getsize(self.path)
        if actual != expected:
            raise MatrixFormatError(
                f"{path}: expected {expected} bytes for {n}x{d} (+{payload_offset} offset), got {actual}")
        self._fd = os.open(self.path, os.O_RDONLY)

    @classmethod
    def open(cls, path, raw: bool = False, n: int | None = None, d: int | None = None,
             page_size: int = DEFAULT_PAGE_SIZE) -> "RowStore":
        """Open a matrix file; header files supply their own shape."""
        if raw:
            if n is None or d is None:
                raise MatrixFormatError("raw files carry no shape; pass n and d explicitly")
            return cls(path, n, d, page_size=page_size)
        hn, hd = read_header(path)
        return cls(path, hn, hd, page_size=page_size, payload_offset=HEADER_SIZE)

    def close(self) -> None:
        if self._fd is not None:
            os.close(self._fd)
            self._fd = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _pread(self, offset: int, size: int) -> bytes:
        return os.pread(self._fd, size, offset)

    def read_pages(self, first_page: int, n_pages: int) -> bytes:
        """Raw bytes of a contiguous page run, truncated at the end of the payload."""
        start = first_page * self.page_size
        end = min((first_page + n_pages) * self.page_size, self.n * self.row_bytes)
        if end <= start:
            return b""
        blob = self._pread(self.payload_offset + start, end - start)
        if len(blob) != end - start:
            raise MatrixFormatError(f"{self.path}: short read at page {first_page} "
                                    f"(wanted {end - start} bytes, got {len(blob)})")
        return blob

    def read_all_into(self, out: np.ndarray, chunk_bytes: int = 64 << 20) -> None:
        """The whole payload into ``out`` (n x d f64, e.g. page-locked), in large reads."""
        view = memoryview(out.reshape(-1).view(np.uint8))
        total = self.n * self.row_bytes
        pos = 0
        while pos < total:
            want = min(chunk_bytes, total - pos)
            got = os.preadv(self._fd, [view[pos:pos + want]], self.payload_offset + pos)
            if got <= 0:
                raise MatrixFormatError(f"{self.path}: short read at byte {pos} of the payload")
            pos += got


def page_runs(ids: np.ndarray, row_bytes: int, page_size: int):
    """Coalesced runs of distinct pages covering ascending row ids (outofcore.py:118-145):
    (runs, total_pages), each run (first_page, n_pages)."""
    ids = np.asarray(ids, dtype=np.int64)
    if ids.size == 0:
        return [], 0
    starts = ids * row_bytes
    first = starts // page_size
    last = (starts + row_bytes - 1) // page_size
    # a new run starts where the next row's first page is past the previous row's last + 1
    brk = np.flatnonzero(first[1:] > last[:-1] + 1) + 1
    lo = np.concatenate(([0], brk))
    hi = np.concatenate((brk - 1, [ids.size - 1]))
    runs = [(int(first[a]), int(last[b]) - int(first[a]) + 1) for a, b in zip(lo, hi)]
    return runs, sum(r[1] for r in runs)


@dataclass
class IoStats:
    """Monotone I/O counters (outofcore.py:148-160)."""

    bytes_requested: int = 0
    bytes_read: int = 0
    cache_hits: int = 0
    cache_misses: int = 0
    rows_elided: int = 0

    def snapshot(self):
        from .engine import IoDelta
        return IoDelta(self.bytes_requested, self.bytes_read, self.cache_hits, self.cache_misses,
                       self.rows_elided)


def fetch_rows(store: RowStore, ids, cache=None, stats: IoStats | None = None) -> np.ndarray:
    """Rows for ascending ids (outofcore.py:163-225): cached rows from ``cache.published``
    (a mapping id -> row), the rest in coalesced page runs.  Host-side helper."""
    ids = np.asarray(ids, dtype=np.int64)
    if ids.size:
        if np.any(np.diff(ids) < 0):
            raise ValueError("row ids must be sorted ascending")
        if ids[0] < 0 or ids[-1] >= store.n:
            bad = ids[0] if ids[0] < 0 else ids[-1]
            raise IndexError(f"row id {int(bad)} out of range [0, {store.n})")
    out = np.empty((ids.size, store.d), dtype=np.float64)
    if stats is not None:
        stats.bytes_requested += store.row_bytes * int(ids.size)
    if ids.size == 0:
        return out
    pos = np.arange(ids.size)
    if cache is not None:
        index = cache.published
        hit = np.fromiter((int(r) in index for r in ids), dtype=bool, count=ids.size)
        for i in np.flatnonzero(hit):
            out[i] = index[int(ids[i])]
        if stats is not None:
            stats.cache_hits += int(hit.sum())
            stats.cache_misses += int((~hit).sum())
        pos = pos[~hit]
    miss = ids[pos]
    runs, total = page_runs(miss, store.row_bytes, store.page_size)
    if stats is not None:
        stats.bytes_read += store.page_size * total
    cur = 0
    for fp, np_ in runs:
        start, stop = fp * store.page_size, (fp + np_) * store.page_size
        flat = np.frombuffer(store.read_pages(fp, np_), dtype="<f8")
        end = cur
        while end < miss.size and miss[end] * store.row_bytes < stop:
            end += 1
        off = (miss[cur:end] * store.row_bytes - start) // 8
        out[pos[cur:end]] = flat[off[:, None] + np.arange(store.d)]
        cur = end
    return out


class RowCache:
    """Host-side form of the reference's partitioned row cache (outofcore.py:228-270),
    for ``fetch_rows`` callers: each partition keeps its smallest ``rows_per_partition``
    collected ids, and the merged index is what ``published`` serves.  (``kmeans_ondisk``
    keeps the same policy in HBM, csrc/sem.cu.)"""

    def __init__(self, n_partitions: int, capacity_bytes: int, row_bytes: int):
        if n_partitions < 1:
            raise ValueError("need at least one partition")
        if capacity_bytes < 0:
            raise ValueError("capacity must be >= 0")
        self.n_partitions = n_partitions
        self.capacity_bytes = capacity_bytes
        self.row_bytes = row_bytes
        self.rows_per_partition = rows_per_partition(capacity_bytes, n_partitions, row_bytes)
        self.partitions: list[dict] = [{} for _ in range(n_partitions)]
        self.published: dict = {}
        self.refresh_count = 0

    def cached_rows(self) -> int:
        return len(self.published)

    def cached_bytes(self) -> int:
        return len(self.published) * self.row_bytes

    def rebuild(self, collected) -> None:
        """Flush, keep each partition's smallest ids from its collected (ids, rows) chunks, publish."""
        merged = {}
        for p in range(self.n_partitions):
            part = {}
            chunks = collected[p]
            if chunks and self.rows_per_partition > 0:
                ids = np.concatenate([np.asarray(c[0], dtype=np.int64) for c in chunks])
                rows = np.concatenate([np.asarray(c[1], dtype=np.float64) for c in chunks], axis=0)
                for i in np.argsort(ids, kind="stable")[: self.rows_per_partition]:
                    part[int(ids[i])] = rows[i].copy()
            self.partitions[p] = part
            merged.update(part)
        self.published = merged
        self.refresh_count += 1


@dataclass(frozen=True)
class CacheSchedule:
    """Refresh at iteration ``start``, then with doubling gaps (outofcore.py:273-279)."""

    start: int = DEFAULT_REFRESH_START

    def __post_init__(self):
        if self.start < 1:
            raise ValueError("refresh start must be >= 1")


def should_refresh(iteration: int, sched: CacheSchedule) -> bool:
    """True at iterations start, 3 start, 7 start, 15 start, ... (outofcore.py:282-290)."""
    if iteration < sched.start or iteration % sched.start != 0:
        return False
    q = iteration // sched.start + 1
    return q & (q - 1) == 0


def rows_per_partition(capacity_bytes: int, T: int, row_bytes: int) -> int:
    """Each worker partition's share of the cache, in rows (RowCache.__init__)."""
    return (capacity_bytes // T) // row_bytes


def load_rows(store: RowStore) -> np.ndarray:
    """The store's payload in host memory (anonymous, so the driver can page-lock and
    map it for the GPU: knb_attach_host_rows)."""
    arr = np.empty((store.n, store.d), dtype=np.float64)
    store.read_all_into(arr)
    return arr


def kmeans_ondisk(store: RowStore, cfg, *, cache_enabled: bool = True,
                  cache_capacity: int = DEFAULT_CACHE_BYTES,
                  schedule: CacheSchedule | None = None, inspect_cache: bool = False):
    """Cluster a file-resident matrix with the rows outside HBM (outofcore.py:440-455).

    Same results as ``kmeans()`` on the same matrix; ``IterationStats.io`` and
    ``KmeansResult.io_totals`` carry the reference's I/O accounting for this run;
    ``inspect_cache`` returns the final HBM cache as ``KmeansResult.row_cache``
    (ids, rows).
    """
    from .engine import _run_sem
    if cfg.mode != "sem":
        raise ValueError("kmeans_ondisk() runs in sem mode; set cfg.mode='sem'")
    cfg.validate()
    if cache_capacity < 0:
        raise ValueError("capacity must be >= 0")
    sched = schedule or CacheSchedule()
    rows = load_rows(store)
    run_cfg = dataclasses.replace(cfg, host_rows=True)
    return _run_sem(rows, run_cfg, dict(T=cfg.T, task_size=cfg.task_size, page_size=store.page_size,
                                        cache_enabled=bool(cache_enabled), cache_capacity=int(cache_capacity),
                                        refresh_start=sched.start, inspect_cache=inspect_cache))
