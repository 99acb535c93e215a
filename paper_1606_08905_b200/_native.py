"""ctypes binding of libknorb200.so (include/knor_b200.h).

There is no CPU fallback: if the library is missing or a CUDA call fails the
error propagates.  Error codes map onto the exception types the reference
raises for the same conditions (ValueError for bad arguments, RuntimeError for
the Sigma counts != n invariant, engine.py:378-380).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KNB_LIB") or os.path.join(HERE, "libknorb200.so")  # KNB_LIB: experiments only

KNB_E_ARG, KNB_E_CUDA, KNB_E_STATE, KNB_E_COUNT, KNB_E_NOMEM = -1, -2, -3, -4, -5
KNB_OPT_MTI_SCAN = 1
MTI_SCAN = {"auto": 0, "exact": 1, "dense": 2, "block": 3, "tc": 4}


class NativeUnavailable(RuntimeError):
    """libknorb200.so is not built (or not loadable); there is no fallback."""


class IterStatsC(ctypes.Structure):
    _fields_ = [
        ("t", ctypes.c_int64),
        ("reassignments", ctypes.c_int64),
        ("wcss", ctypes.c_double),
        ("dist_comps", ctypes.c_int64),
        ("skips", ctypes.c_int64),
        ("pruned_stale", ctypes.c_int64),
        ("pruned_tight", ctypes.c_int64),
        ("converged", ctypes.c_int32),
        ("stop", ctypes.c_int32),
        ("count_total", ctypes.c_int64),
    ]


_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_D = ctypes.c_double
_PI32 = ctypes.POINTER(ctypes.c_int32)
_PI64 = ctypes.POINTER(ctypes.c_int64)
_PD = ctypes.POINTER(ctypes.c_double)

# name -> argtypes (all return int status except knb_last_error / knb_version)
SIGNATURES = {
    "knb_device_info": [ctypes.c_int, _PI32, _PI64, _PI32, _PI32],
    "knb_create": [ctypes.c_int, _I64, _I64, _I64, _I32, _I32, _I32, _I32, _D, _P, ctypes.POINTER(_P)],
    "knb_destroy": [_P],
    "knb_release_memory": [ctypes.c_int],
    "knb_upload_rows": [_P, _P, _I64, _I64],
    "knb_attach_rows": [_P, _P],
    "knb_attach_host_rows": [_P, _P],
    "knb_sem_configure": [_P, _I32, _I64, _I64, _I32, _I64, _I32],
    "knb_sem_io": [_P, _PI64, _I32],
    "knb_sem_cache": [_P, _PI64, _P, _I64, _PI64],
    "knb_upload_rows_f32": [_P, _P, _I64, _I64],
    "knb_attach_rows_f32": [_P, _P],
    "knb_tc_info": [_P, _PI32, _PI64, _PI64],
    "knb_tc_scores": [_P, _P, _PD],
    "knb_check_finite": [_P, _PI64],
    "knb_exchange_len": [_P, _PI64],
    "knb_set_exchange": [_P, _P, _I64],
    "knb_exchange_ptr": [_P, ctypes.POINTER(_P)],
    "knb_set_centroids": [_P, _P],
    "knb_init_gather": [_P, _P, _I32],
    "knb_init_from_exchange": [_P, _I32, _I32],
    "knb_init_partition_local": [_P, _P],
    "knb_init_partition_finish": [_P],
    "knb_kpp_update": [_P, _I32, _PD],
    "knb_kpp_psum": [_P, _D, _PD],
    "knb_kpp_search": [_P, _D, _D, _PI64],
    "knb_kpp_release": [_P],
    "knb_kpp_run": [_P, _I64, _P, _I32, _P, _PI32],
    "knb_iter_local": [_P],
    "knb_iter_finish": [_P],
    "knb_iterate": [_P, ctypes.POINTER(IterStatsC)],
    "knb_run": [_P, _I32, _PI32],
    "knb_enqueue": [_P, _I32],
    "knb_validate": [_P, _PI64, _PI64],
    "knb_get_stats": [_P, ctypes.POINTER(IterStatsC), _I32, _PI32],
    "knb_get_state": [_P, _PI32, _PI32, _PI64, _PI32],
    "knb_get_centroids": [_P, _P, _P, _P, _P],
    "knb_get_assignments": [_P, _P, _I64, _I64],
    "knb_get_bounds": [_P, _P, _P],
    "knb_sync": [_P],
    "knb_set_ignore_stop": [_P, _I32],
    "knb_set_stream": [_P, _P],
    "knb_state_bytes": [_P, _PI64],
    "knb_describe": [_P, _PI32, _PI32, _PI32, _PI32],
    "knb_mti_tc_info": [_P, _PI32, _PI64],
    "knb_mti_tc_scores": [_P, _P],
    "knb_mti_tc_prof": [_PI64, _PI32],
    "knb_staging_reserve": [ctypes.c_int],
    "knb_measure_peaks": [ctypes.c_int, _PD, _PD],
    "knb_block_distances": [ctypes.c_int, _P, _I64, _P, _I32, _I32, _P, _P, _P],
    "knb_rowwise": [ctypes.c_int, _P, _I64, _P, _I32, _I32, _I32, _P],
    "knb_set_option": [_P, _I32, _I64],
    "knb_fill_uniform_pcg64": [_P, _I64, _I64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, _P],
}

_lib = None


def lib():
    """Load the in-tree library (raises NativeUnavailable, never falls back)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeUnavailable(
            f"{LIB_PATH} is not built; run `python -m paper_1606_08905_b200.build` "
            "(nvcc, sm_100a). There is no CPU fallback.")
    try:
        h = ctypes.CDLL(LIB_PATH)
    except OSError as exc:  # pragma: no cover - depends on the host
        raise NativeUnavailable(f"cannot load {LIB_PATH}: {exc}") from exc
    h.knb_version.restype = ctypes.c_int
    h.knb_version.argtypes = []
    h.knb_last_error.restype = ctypes.c_char_p
    h.knb_last_error.argtypes = []
    h.knb_f32_supported.restype = ctypes.c_int
    h.knb_f32_supported.argtypes = [_I32, _I32, _I32]
    h.knb_mti_compact_ok.restype = ctypes.c_int
    h.knb_mti_compact_ok.argtypes = [_I64]
    for name, args in SIGNATURES.items():
        fn = getattr(h, name)
        fn.restype = ctypes.c_int
        fn.argtypes = args
    _lib = h
    return h


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = lib().knb_last_error().decode(errors="replace")
    if rc == KNB_E_ARG:
        raise ValueError(msg)
    if rc == KNB_E_NOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def ptr(a: np.ndarray) -> ctypes.c_void_p:
    return ctypes.c_void_p(a.ctypes.data)


class Context:
    """One GPU shard: owns a knb_ctx and frees it on close()."""

    def __init__(self, device: int, n_global: int, n_local: int, row_lo: int, d: int, k: int,
                 pruning: bool, max_iters: int, tolerance: float, stream: int | None = None):
        self.L = lib()
        self.device = device
        self.n_local, self.d, self.k = n_local, d, k
        self.max_iters = max_iters
        h = ctypes.c_void_p()
        check(self.L.knb_create(device, n_global, n_local, row_lo, d, k, int(bool(pruning)),
                                max_iters, float(tolerance), ctypes.c_void_p(stream or 0), ctypes.byref(h)))
        self.h = h

    # lifetime
    def close(self) -> None:
        if getattr(self, "h", None):
            self.L.knb_destroy(self.h)
            self.h = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # rows
    def upload(self, rows: np.ndarray, lo: int = 0) -> None:
        rows = np.ascontiguousarray(rows, dtype=np.float64)
        check(self.L.knb_upload_rows(self.h, ptr(rows), lo, rows.shape[0]))
        self.sync()  # the caller may release the host buffer

    def upload_async(self, rows: np.ndarray, lo: int = 0) -> None:
        """Caller guarantees `rows` (ideally pinned) outlives the copy (sync before reuse)."""
        check(self.L.knb_upload_rows(self.h, ptr(rows), lo, rows.shape[0]))

    def attach(self, dev_ptr: int) -> None:
        check(self.L.knb_attach_rows(self.h, ctypes.c_void_p(dev_ptr)))

    def attach_host(self, rows: np.ndarray) -> None:
        """Rows stay in host memory (page-locked + mapped) and are read over the host link.
        A file mapping the driver cannot lock (np.memmap) is first read into anonymous
        memory -- still no HBM copy."""
        rows = np.ascontiguousarray(rows, dtype=np.float64)
        try:
            check(self.L.knb_attach_host_rows(self.h, ptr(rows)))
        except RuntimeError:
            if not isinstance(rows, np.memmap) and rows.base is None:
                raise
            rows = np.array(rows, dtype=np.float64, order="C")
            check(self.L.knb_attach_host_rows(self.h, ptr(rows)))
        self._host_rows = rows  # the registered buffer lives as long as the context

    def sem_configure(self, T: int, task_size: int, page_size: int, cache_enabled: bool,
                      cache_capacity: int, refresh_start: int) -> None:
        check(self.L.knb_sem_configure(self.h, T, task_size, page_size, 1 if cache_enabled else 0,
                                       cache_capacity, refresh_start))

    def sem_io(self, count: int) -> np.ndarray:
        """(count, 5) int64: bytes_requested, bytes_read, cache_hits, cache_misses, rows."""
        out = np.zeros((max(count, 1), 5), dtype=np.int64)
        check(self.L.knb_sem_io(self.h, out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), count))
        return out[:count]

    def sem_cache(self, with_rows: bool = True):
        """(ids, rows) of the published HBM row cache."""
        cnt = ctypes.c_int64()
        check(self.L.knb_sem_cache(self.h, None, None, 0, ctypes.byref(cnt)))
        m = cnt.value
        ids = np.zeros(max(m, 1), dtype=np.int64)
        rows = np.zeros((max(m, 1), self.d), dtype=np.float64) if with_rows else None
        check(self.L.knb_sem_cache(self.h, ids.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                   ptr(rows) if with_rows else None, m, ctypes.byref(cnt)))
        return ids[:m], (rows[:m] if with_rows else None)

    def upload_f32(self, rows: np.ndarray, lo: int = 0) -> None:
        """f32 rows for the tensor-core path (see f32_supported)."""
        rows = np.ascontiguousarray(rows, dtype=np.float32)
        check(self.L.knb_upload_rows_f32(self.h, ptr(rows), lo, rows.shape[0]))
        self.sync()

    def upload_f32_async(self, rows: np.ndarray, lo: int = 0) -> None:
        check(self.L.knb_upload_rows_f32(self.h, ptr(rows), lo, rows.shape[0]))

    def attach_f32(self, dev_ptr: int) -> None:
        check(self.L.knb_attach_rows_f32(self.h, ctypes.c_void_p(dev_ptr)))

    def tc_scores(self, dev_ptr: int) -> float:
        """Dump the tensor-core scores (n_local x k_pad f32) into device memory at
        ``dev_ptr``; returns the certificate's relative error e."""
        e = ctypes.c_double()
        check(self.L.knb_tc_scores(self.h, ctypes.c_void_p(dev_ptr), ctypes.byref(e)))
        return float(e.value)

    def tc_info(self) -> dict:
        a = ctypes.c_int32()
        f, g = ctypes.c_int64(), ctypes.c_int64()
        check(self.L.knb_tc_info(self.h, ctypes.byref(a), ctypes.byref(f), ctypes.byref(g)))
        return dict(active=bool(a.value), flagged_rows=int(f.value), full_reranks=int(g.value))

    def first_nonfinite_row(self) -> int:
        v = ctypes.c_int64()
        check(self.L.knb_check_finite(self.h, ctypes.byref(v)))
        return int(v.value)

    # exchange
    def exchange_len(self) -> int:
        v = ctypes.c_int64()
        check(self.L.knb_exchange_len(self.h, ctypes.byref(v)))
        return int(v.value)

    def set_exchange(self, dev_ptr: int, length: int) -> None:
        check(self.L.knb_set_exchange(self.h, ctypes.c_void_p(dev_ptr), length))

    # init
    def set_centroids(self, means: np.ndarray) -> None:
        means = np.ascontiguousarray(means, dtype=np.float64)
        check(self.L.knb_set_centroids(self.h, ptr(means)))

    def init_gather(self, ids) -> None:
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        check(self.L.knb_init_gather(self.h, ptr(ids), ids.shape[0]))

    def init_from_exchange(self, first: int, count: int) -> None:
        check(self.L.knb_init_from_exchange(self.h, first, count))

    def init_partition_local(self, labels: np.ndarray) -> None:
        labels = np.ascontiguousarray(labels, dtype=np.int32)
        check(self.L.knb_init_partition_local(self.h, ptr(labels)))

    def init_partition_finish(self) -> None:
        check(self.L.knb_init_partition_finish(self.h))

    def kpp_update(self, first: bool) -> float:
        v = ctypes.c_double()
        check(self.L.knb_kpp_update(self.h, int(first), ctypes.byref(v)))
        return float(v.value)

    def kpp_psum(self, total: float) -> float:
        v = ctypes.c_double()
        check(self.L.knb_kpp_psum(self.h, float(total), ctypes.byref(v)))
        return float(v.value)

    def kpp_search(self, total: float, threshold: float) -> int:
        v = ctypes.c_int64()
        check(self.L.knb_kpp_search(self.h, float(total), float(threshold), ctypes.byref(v)))
        return int(v.value)

    def kpp_run(self, first_pick: int, u: np.ndarray) -> tuple[list[int], bool]:
        """Single-GPU kmeans++ on the device; returns (picks, degenerate)."""
        u = np.ascontiguousarray(u, dtype=np.float64)
        picks = np.empty(self.k, dtype=np.int64)
        deg = ctypes.c_int32()
        check(self.L.knb_kpp_run(self.h, int(first_pick), ptr(u) if u.size else None, self.k, ptr(picks),
                                 ctypes.byref(deg)))
        return [int(p) for p in picks], bool(deg.value)

    def kpp_release(self) -> None:
        check(self.L.knb_kpp_release(self.h))

    # iterations
    def iter_local(self) -> None:
        check(self.L.knb_iter_local(self.h))

    def iter_finish(self) -> None:
        check(self.L.knb_iter_finish(self.h))

    def iterate(self) -> IterStatsC:
        s = IterStatsC()
        check(self.L.knb_iterate(self.h, ctypes.byref(s)))
        return s

    def run(self, batch: int) -> int:
        v = ctypes.c_int32()
        check(self.L.knb_run(self.h, batch, ctypes.byref(v)))
        return int(v.value)

    def enqueue(self, count: int) -> None:
        """Queue ``count`` iterations (graph replays after the first); no host sync."""
        check(self.L.knb_enqueue(self.h, count))

    def validate(self) -> tuple[int, int]:
        a, b = ctypes.c_int64(), ctypes.c_int64()
        check(self.L.knb_validate(self.h, ctypes.byref(a), ctypes.byref(b)))
        return int(a.value), int(b.value)

    # results
    def stats(self) -> list[IterStatsC]:
        buf = (IterStatsC * self.max_iters)()
        cnt = ctypes.c_int32()
        check(self.L.knb_get_stats(self.h, buf, self.max_iters, ctypes.byref(cnt)))
        return [buf[i] for i in range(cnt.value)]

    def state(self) -> dict:
        stop, conv, err = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        t = ctypes.c_int64()
        check(self.L.knb_get_state(self.h, ctypes.byref(stop), ctypes.byref(conv), ctypes.byref(t),
                                   ctypes.byref(err)))
        return dict(stop=bool(stop.value), converged=bool(conv.value), t=int(t.value), count_error=bool(err.value))

    def centroids(self):
        means = np.empty((self.k, self.d))
        prev = np.empty((self.k, self.d))
        counts = np.empty(self.k, dtype=np.int64)
        drift = np.empty(self.k)
        check(self.L.knb_get_centroids(self.h, ptr(means), ptr(prev), ptr(counts), ptr(drift)))
        return means, prev, counts, drift

    def assignments(self, lo: int = 0, count: int | None = None, out: np.ndarray | None = None) -> np.ndarray:
        count = self.n_local - lo if count is None else count
        if out is None:
            out = np.empty(count, dtype=np.int32)
        check(self.L.knb_get_assignments(self.h, ptr(out), lo, count))
        return out

    def bounds(self):
        u = np.empty(self.n_local)
        t = np.empty(self.n_local, dtype=np.uint8)
        check(self.L.knb_get_bounds(self.h, ptr(u), ptr(t)))
        return u, t.astype(bool)

    def sync(self) -> None:
        check(self.L.knb_sync(self.h))

    def set_stream(self, stream: int | None) -> None:
        check(self.L.knb_set_stream(self.h, ctypes.c_void_p(stream or 0)))

    def set_ignore_stop(self, on: bool) -> None:
        check(self.L.knb_set_ignore_stop(self.h, int(on)))

    def set_option(self, option: int, value: int) -> None:
        check(self.L.knb_set_option(self.h, option, value))

    def state_bytes(self) -> int:
        v = ctypes.c_int64()
        check(self.L.knb_state_bytes(self.h, ctypes.byref(v)))
        return int(v.value)

    def mti_tc_info(self) -> dict:
        a, u = ctypes.c_int32(), ctypes.c_int64()
        check(self.L.knb_mti_tc_info(self.h, ctypes.byref(a), ctypes.byref(u)))
        return dict(available=bool(a.value), uncertified=int(u.value))

    def mti_tc_scores(self, dev_ptr: int) -> None:
        """Scores D~ (n_local x N f32, N = k rounded up to 16) of the tcgen05 MTI pass."""
        check(self.L.knb_mti_tc_scores(self.h, ctypes.c_void_p(dev_ptr)))

    def describe(self) -> dict:
        a, b, c, d = (ctypes.c_int32() for _ in range(4))
        check(self.L.knb_describe(self.h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c), ctypes.byref(d)))
        return dict(dense_dp=a.value, tma=bool(b.value), grid_dense=c.value,
                    grid_mti=abs(d.value), mti_kernel="tensor-core" if d.value < 0 else "exact-scan")


def f32_supported(d: int, k: int, pruning: bool) -> bool:
    """Whether f32 rows stay f32 on the device (dense tcgen05 path); else they are upcast."""
    return bool(lib().knb_f32_supported(int(d), int(k), int(bool(pruning))))


def mti_compact_ok(n_local: int) -> bool:
    """Whether a shard of n_local rows may run the compacted MTI kernel (32-bit row
    indices); larger shards run the block-dense MTI pass (same results)."""
    return bool(lib().knb_mti_compact_ok(int(n_local)))


def release_memory(device: int = 0) -> None:
    """Return the device memory the library's pool holds but no context uses to the driver
    (the pool keeps it between kmeans() calls, as torch's caching allocator does)."""
    check(lib().knb_release_memory(int(device)))


def reserve_staging(device: int = 0) -> None:
    """Allocate the pinned staging pool for large host transfers now (otherwise the first
    large kmeans() call of the process pays for pinning it)."""
    check(lib().knb_staging_reserve(int(device)))


def mti_tc_prof() -> tuple[bool, list[int]]:
    """(enabled, 16 cycle counters) of a -DKNB_TCX_PROF=1 build; read and cleared."""
    out = (ctypes.c_int64 * 16)()
    en = ctypes.c_int32()
    check(lib().knb_mti_tc_prof(out, ctypes.byref(en)))
    return bool(en.value), [int(v) for v in out]


def device_info(device: int = 0) -> dict:
    sms, cmaj, cmin = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    hbm = ctypes.c_int64()
    check(lib().knb_device_info(device, ctypes.byref(sms), ctypes.byref(hbm), ctypes.byref(cmaj), ctypes.byref(cmin)))
    return dict(sms=sms.value, hbm_bytes=hbm.value, cc=(cmaj.value, cmin.value))


def measure_peaks(device: int = 0) -> dict:
    """FP64 FMA rate and device copy bandwidth measured on `device` (roofline denominators)."""
    f, c = ctypes.c_double(), ctypes.c_double()
    check(lib().knb_measure_peaks(device, ctypes.byref(f), ctypes.byref(c)))
    return dict(dfma_per_s=f.value, copy_bytes_per_s=c.value)
