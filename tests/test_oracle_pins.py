"""Pin the CPU oracle before trusting it (CPU only).

1. oracle.lloyd vs the golden fixtures produced by the REFERENCE package
   (oracle/make_golden.py): bit-identical assignment history, per-iteration
   counters and centroids.
2. The reference's own known-answer vectors (3-4-5, tie -> lowest id, hand
   example, geometry hand values, MTI hand trace, inflate semantics).
3. oracle/exact_tree.c (the contraction tree the GPU's exact recipe follows)
   vs np.vecdot on this host -- skipped at the bit level when the host BLAS
   picks another kernel.
4. When /root/reference is mounted: oracle vs the live reference.
"""

from __future__ import annotations

import ctypes
import hashlib
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT, golden
from oracle import lloyd as O
from oracle.golden_cases import CASES, case_cfg, case_data


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int32).tobytes()).hexdigest()


def _run_oracle(name, collect=True):
    c = case_cfg(name)
    k = c.pop("k")
    return O.lloyd(case_data(name), k, init=c.pop("init", "forgy"), initial=c.pop("initial", None),
                   collect=collect, threads=4, **c)


@pytest.mark.parametrize("name", list(CASES))
def test_oracle_matches_reference_golden(name):
    g = golden(name)
    r = _run_oracle(name)
    assert [_sha(h) for h in r.history] == list(g["history_sha"])
    for key in ("reassignments", "dist_comps", "skips", "pruned_stale", "pruned_tight"):
        assert np.array_equal(np.array([getattr(s, key) for s in r.iterations]), g[key]), key
    assert np.array_equal(r.means, g["means"])
    assert np.array_equal(r.prev_means, g["prev_means"])
    assert np.array_equal(r.counts, g["counts"])
    assert np.array_equal(r.init_means, g["init_means"])
    assert np.array_equal(r.assignments, g["assignments"].astype(np.int32))
    assert bool(r.converged) == bool(g["converged"])
    np.testing.assert_allclose([s.wcss for s in r.iterations], g["wcss"], rtol=1e-12)


def test_known_answers():
    # distance.py / test_distance.py:18-19, :59-62
    assert float(O.dist_to(np.array([[0.0, 0.0]]), np.array([3.0, 4.0]))[0]) == 5.0
    ids, best = O.nearest(np.array([[0.0]]), np.array([[-1.0], [1.0]]))
    assert ids[0] == 0 and best[0] == 1.0
    # hand example (test_engine.py:10-22)
    r = O.lloyd(np.array([[0.0], [1.0], [10.0], [11.0]]), 2, init="given",
                initial=np.array([[0.0], [10.0]]), pruning=False, max_iters=20)
    assert r.n_iterations == 2 and r.converged
    assert r.assignments.tolist() == [0, 0, 1, 1]
    assert np.allclose(r.means, [[0.5], [10.5]])
    # geometry of {0, 2, 6} (test_pruning.py:36-43)
    half, hmin = O.half_geometry(np.array([[0.0], [2.0], [6.0]]))
    assert half[0, 1] == 1.0 and half[0, 2] == 3.0 and half[1, 2] == 2.0
    assert hmin.tolist() == [1.0, 1.0, 2.0]
    # MTI hand trace (test_pruning.py:101-117)
    half, _ = O.half_geometry(np.array([[0.0], [6.0], [100.0]]))
    a, u, t = np.array([0], np.int32), np.array([5.0]), np.array([False])
    ctr = dict(skips=0, pruned_stale=0, pruned_tight=0, computed=0)
    O.mti_scan(np.array([[5.0]]), np.array([[0.0], [6.0], [100.0]]), half, a, u, t, ctr)
    assert a[0] == 1 and u[0] == 1.0 and t[0]
    assert ctr["computed"] == 2 and ctr["pruned_stale"] + ctr["pruned_tight"] == 1
    # k = 1 geometry never blocks a skip (test_pruning.py:25-33)
    _, hmin = O.half_geometry(np.array([[5.0]]))
    assert hmin[0] == np.inf


def _tree_lib():
    so = os.path.join(ROOT, "oracle", "liboracle_tree.so")
    if not os.path.exists(so):
        subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "oracle")])
    return ctypes.CDLL(so)


@pytest.mark.parametrize("d", [1, 3, 8, 15, 16, 17, 31, 32, 33, 48, 64, 65, 100, 256])
def test_exact_tree_restatement_matches_host_vecdot(d):
    lib = _tree_lib()
    rng = np.random.default_rng(d)
    rows = rng.normal(size=(3000, d)) * rng.uniform(0.1, 50)
    ref = rng.normal(size=d)
    out = np.empty(3000)
    lib.oracle_tree_sqdist(rows.ctypes.data_as(ctypes.c_void_p), ref.ctypes.data_as(ctypes.c_void_p),
                           ctypes.c_int64(3000), ctypes.c_int(d), ctypes.c_int(0),
                           out.ctypes.data_as(ctypes.c_void_p))
    want = O.sq_to(rows, ref)
    np.testing.assert_allclose(out, want, rtol=1e-13)
    arch = _blas_arch()
    if "SkylakeX" in arch or "Cooperlake" in arch or "SapphireRapids" in arch:
        assert np.array_equal(out, want), f"tree model differs bitwise on {arch}"


def _blas_arch():
    import io
    from contextlib import redirect_stdout
    buf = io.StringIO()
    with redirect_stdout(buf):
        np.show_runtime()
    return buf.getvalue()


REF = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted")
@pytest.mark.parametrize("name", ["mix_pruned", "kpp_pruned", "d17_pruned", "rp_dense"])
def test_oracle_matches_live_reference_multithreaded(name):
    import sys
    sys.path.insert(0, REF)
    try:
        from numakmeans import EngineConfig, kmeans
    finally:
        sys.path.remove(REF)
    c = case_cfg(name)
    m = case_data(name)
    ref = kmeans(m, EngineConfig(k=c["k"], init=c.get("init", "forgy"), seed=c.get("seed", 0), T=4,
                                 pruning=c.get("pruning", True), max_iters=c.get("max_iters", 100),
                                 collect_assignments=True, task_size=257))
    mine = O.lloyd(m, c["k"], init=c.get("init", "forgy"), seed=c.get("seed", 0), T=4, task_size=257,
                   pruning=c.get("pruning", True), max_iters=c.get("max_iters", 100), collect=True, threads=3)
    assert mine.n_iterations == ref.n_iterations
    for a, b in zip(mine.history, ref.assignment_history):
        assert np.array_equal(a, b)
    assert np.array_equal(mine.means, ref.centroids.means)
