"""The reference's public primitives, computed on the GPU with the engine's recipe.

    euclidean_distance, rowwise_distances, block_distances, row_sqnorms,
    nearest_centroid                       numakmeans distance.py:19-82
    CentroidGeometry, centroid_geometry    numakmeans pruning.py:33-61
    init_centroids                         numakmeans centroids.py:131-189

Every distance is the exact f64 recipe (exact subtract, the OpenBLAS ddot tree,
sqrt) that ``kmeans()`` uses, so these agree bit for bit with the engine and the
reference; ties in ``nearest_centroid`` go to the lowest id.  They run through the
C ABI (``knb_block_distances`` / ``knb_rowwise``; ``init_centroids`` through a
context and the device init) -- there is no CPU implementation to fall back to.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from .centroids import CentroidSet, device_init
from .matrix import check_shape
from .parallel import LocalComm


def _device() -> int:
    try:
        import torch
        return torch.cuda.current_device() if torch.cuda.is_available() else 0
    except Exception:  # noqa: BLE001
        return 0


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def euclidean_distance(a, b) -> float:
    """Distance between two equal-length vectors (distance.py:19-25)."""
    a, b = _f64(a), _f64(b)
    if a.shape != b.shape or a.ndim != 1:
        raise ValueError(f"length mismatch: {a.shape} vs {b.shape}")
    return float(rowwise_distances(a[None, :], b)[0])


def rowwise_distances(rows, refs, buf=None, out=None) -> np.ndarray:
    """Row i of ``rows`` vs row i of ``refs``, or one shared ref vector (distance.py:36-39)."""
    rows, refs = _f64(rows), _f64(refs)
    m, d = rows.shape
    shared = refs.ndim == 1
    if (shared and refs.shape[0] != d) or (not shared and refs.shape != rows.shape):
        raise ValueError(f"shape mismatch: {rows.shape} vs {refs.shape}")
    res = np.empty(m) if out is None else out
    _native.check(_native.lib().knb_rowwise(_device(), _native.ptr(rows), m, _native.ptr(refs), int(shared), d, 1,
                                            _native.ptr(res)))
    return res


def block_distances(rows, centroids, buf=None, out=None) -> np.ndarray:
    """Full (m, k) distance matrix (distance.py:42-63); ``buf`` is accepted and unused."""
    rows, centroids = _f64(rows), _f64(centroids)
    if rows.ndim != 2 or centroids.ndim != 2 or rows.shape[1] != centroids.shape[1]:
        raise ValueError(f"shape mismatch: {rows.shape} vs {centroids.shape}")
    m, d = rows.shape
    k = centroids.shape[0]
    res = np.empty((m, k)) if out is None else out
    _native.check(_native.lib().knb_block_distances(_device(), _native.ptr(rows), m, _native.ptr(centroids), k, d,
                                                    _native.ptr(res), None, None))
    return res


def row_sqnorms(rows) -> np.ndarray:
    """Squared L2 norm of each row with the kernels' contraction (distance.py:66-72)."""
    rows = _f64(rows)
    m, d = rows.shape
    res = np.empty(m)
    _native.check(_native.lib().knb_rowwise(_device(), _native.ptr(rows), m, None, 0, d, 0, _native.ptr(res)))
    return res


def nearest_centroid(rows, centroids):
    """Nearest-centroid ids (int32) and distances; ties to the lowest id (distance.py:75-82)."""
    rows, centroids = _f64(rows), _f64(centroids)
    if rows.ndim != 2 or centroids.ndim != 2 or rows.shape[1] != centroids.shape[1]:
        raise ValueError(f"shape mismatch: {rows.shape} vs {centroids.shape}")
    m, d = rows.shape
    k = centroids.shape[0]
    ids = np.empty(m, dtype=np.int32)
    best = np.empty(m)
    _native.check(_native.lib().knb_block_distances(_device(), _native.ptr(rows), m, _native.ptr(centroids), k, d,
                                                    None, _native.ptr(ids), _native.ptr(best)))
    return ids, best


@dataclass
class CentroidGeometry:
    """Pairwise half-distances between centroids and per-centroid row minima (pruning.py:33-45)."""

    half_dist: np.ndarray  # (k, k) symmetric, zero diagonal
    half_min: np.ndarray   # (k,)

    def state_bytes(self) -> int:
        return self.half_dist.nbytes + self.half_min.nbytes


def centroid_geometry(c: CentroidSet) -> CentroidGeometry:
    """half_dist[a, b] = d(c_a, c_b) / 2 and half_min[a] = min over b != a (pruning.py:48-61).
    The subtract's sign cannot change a square, so the device's pairwise matrix is exactly
    the reference's per-row computation."""
    means = _f64(c.means)
    k = means.shape[0]
    half = block_distances(means, means) * 0.5
    np.fill_diagonal(half, 0.0)
    if k == 1:
        half_min = np.array([np.inf])
    else:
        half_min = (half + np.diag(np.full(k, np.inf))).min(axis=1)
    return CentroidGeometry(half_dist=half, half_min=half_min)


def init_centroids(m, k: int, method: str = "forgy", seed: int = 0, initial=None) -> CentroidSet:
    """Seeded initial centroids (centroids.py:131-189) by the engine's device init: the
    host draws the reference's RNG stream, the device does every pass over the rows."""
    from .centroids import INIT_METHODS
    if method not in INIT_METHODS:
        raise ValueError(f"unknown init method {method!r}")
    if k < 1:
        raise ValueError("k must be >= 1")
    rows = check_shape(m)
    n, d = rows.shape
    ctx = _native.Context(_device(), n, n, 0, d, k, False, 1, 0.0, None)
    try:
        ctx.upload(rows)
        bad = ctx.first_nonfinite_row()
        if bad >= 0:
            from .matrix import MatrixFormatError
            raise MatrixFormatError(f"non-finite value in row {bad}")
        device_init(ctx, LocalComm(), None, method, k, seed, initial, n, 0, n, d)
        means, _, _, _ = ctx.centroids()
    finally:
        ctx.close()
    return CentroidSet.from_means(means)
