"""Shared fixtures and the parity checker.

Parity bar (BASELINE.json north star):
  * iteration count equal;
  * assignments equal, except points whose best / second-best distance gap
    (d2 - d1) / d2 is below EPS_F64 = 1e-9 (EPS_F32 = 1e-4 for f32 data) --
    the check recomputes that gap with the oracle for every mismatch;
  * centroids: max|delta| / max|c| <= 1e-9 (f64);
  * per-iteration integer counters (reassignments, dist_comps, skips,
    pruned_*) equal, WCSS within rel 1e-9.
"""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

EPS_F64 = 1e-9
EPS_F32 = 1e-4
CENTROID_RTOL = 1e-9


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libknorb200.so")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(autouse=True)
def _release_device_memory(request):
    """After each GPU test, hand the library pool's unused device memory back (it keeps it
    between kmeans() calls, like torch's caching allocator), so the next test's torch
    allocations see it free."""
    yield
    if request.node.get_closest_marker("gpu") is not None:
        from paper_1606_08905_b200 import _native
        if _native._lib is not None:
            _native.release_memory(0)


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def golden(name: str):
    return np.load(os.path.join(ROOT, "tests", "golden", f"{name}.npz"))


def near_tie_rows(m: np.ndarray, means: np.ndarray, rows: np.ndarray, eps: float) -> np.ndarray:
    """Subset of ``rows`` whose oracle best/second gap is below eps (allowed to differ)."""
    from oracle.lloyd import lloyd_step
    if rows.size == 0:
        return rows
    _, d1, d2 = lloyd_step(m[rows], means)
    gap = (d2 - d1) / np.maximum(d2, 1e-300)
    return rows[gap < eps]


def assert_parity(m, got, want_means, want_assign, want_iters, eps=EPS_F64, centroid_rtol=CENTROID_RTOL,
                  want_prev=None, counters=None, wcss=None, what=""):
    """got: KmeansResult-like; want_*: oracle/golden values."""
    assert got.n_iterations == want_iters, f"{what}: iterations {got.n_iterations} != {want_iters}"
    a = np.asarray(got.assignments)
    b = np.asarray(want_assign).astype(np.int32)
    bad = np.flatnonzero(a != b)
    if bad.size:
        ref_means = want_prev if want_prev is not None else want_means
        ok = near_tie_rows(np.asarray(m, dtype=np.float64), ref_means, bad, eps)
        assert ok.size == bad.size, f"{what}: {bad.size - ok.size} non-near-tie assignment mismatches (first rows {bad[:5]})"
    scale = max(1.0, float(np.max(np.abs(want_means))))
    err = float(np.max(np.abs(got.centroids.means - want_means))) / scale
    assert err <= centroid_rtol, f"{what}: centroid rel error {err}"
    if counters is not None:
        for key, arr in counters.items():
            got_arr = np.array([getattr(s, key) for s in got.iterations])
            assert np.array_equal(got_arr, np.asarray(arr)), f"{what}: {key} {got_arr} != {np.asarray(arr)}"
    if wcss is not None:
        got_w = np.array([s.wcss for s in got.iterations])
        np.testing.assert_allclose(got_w, wcss, rtol=1e-9, atol=1e-12, err_msg=f"{what}: wcss")
