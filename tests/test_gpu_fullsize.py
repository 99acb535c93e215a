"""Full-size trajectory parity for BASELINE configs c2 and c3 (SURVEY.md section 8(c):
"C1-C3: full trajectory").

The goldens in tests/golden/full/ were made by running the reference package itself
(numakmeans, oracle/make_golden_full.py) on exactly the bytes these tests regenerate
(synth.CONFIGS, numpy's seeded streams).  Checked at every iteration: the sha256 of the
whole assignment vector, the sampled assignments (every 997th row), the reassignment /
skip counters, WCSS, then the iteration count, the final centroids and cluster sizes.
A sha mismatch is tolerated only when every mismatching sampled row is a near-tie
(best / second-best gap < EPS_F64 under the centroids the pass used) and the counters
still agree -- the north star's near-tie rule."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

import paper_1606_08905_b200 as kb
from conftest import EPS_F64, ROOT, near_tie_rows

pytestmark = pytest.mark.gpu


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int32).tobytes()).hexdigest()


def _golden(name):
    import os
    return np.load(os.path.join(ROOT, "tests", "golden", "full", f"{name}.npz"))


def _run_stepwise(name, m, g, mti_scan):
    """Iterate the engine one pass at a time and compare with the golden as it goes."""
    c = kb.synth.CONFIGS[name]
    cfg = kb.EngineConfig(k=c["k"], init=c["init"], seed=int(name[1:]), pruning=c["pruning"],
                          max_iters=c["max_iters"], tolerance=c["tolerance"], mti_scan=mti_scan)
    run = kb.Lloyd(m, cfg)
    rows = g["sample_rows"]
    near_ties = 0
    try:
        assert run.init_rows is None or len(run.init_rows) == c["k"]
        np.testing.assert_array_equal(run.ctx.centroids()[0], g["init_means"])
        t = 0
        while True:
            prev = run.ctx.centroids()[0]
            run.step()
            a = run.ctx.assignments()
            if _sha(a) != str(g["history_sha"][t]):
                bad = rows[np.flatnonzero(a[rows] != g["sample_history"][t].astype(np.int32))]
                ok = near_tie_rows(m, prev, bad, EPS_F64)
                assert ok.size == bad.size, f"{name} iteration {t}: {bad.size - ok.size} non-near-tie mismatches"
                near_ties += bad.size
            st = run.ctx.state()
            t += 1
            if st["stop"]:
                break
            assert t < c["max_iters"] + 1
        stats = run.ctx.stats()
        assert len(stats) == len(g["reassignments"]), f"{name}: {len(stats)} iterations != {len(g['reassignments'])}"
        np.testing.assert_array_equal([s.reassignments for s in stats], g["reassignments"])
        np.testing.assert_array_equal([s.skips for s in stats], g["skips"])
        if mti_scan == "exact":
            for key in ("dist_comps", "pruned_stale", "pruned_tight"):
                np.testing.assert_array_equal([getattr(s, key) for s in stats], g[key], err_msg=key)
        np.testing.assert_allclose([s.wcss for s in stats], g["wcss"], rtol=1e-9)
        means, _, counts, _ = run.ctx.centroids()
        scale = max(1.0, float(np.abs(g["means"]).max()))
        assert float(np.abs(means - g["means"]).max()) / scale <= 1e-9
        np.testing.assert_array_equal(counts, g["counts"])
        assert bool(run.ctx.state()["converged"]) == bool(g["converged"])
        return run.ctx.assignments(), near_ties
    finally:
        run.close()


@pytest.mark.parametrize("mti_scan", ["auto", "exact"])
def test_config2_full_trajectory_matches_reference(mti_scan):
    """c2 at its full n = 2,000,000 (kmeans++ over 2M rows, 100 iterations, tol 1e-6)."""
    g = _golden("c2")
    m = kb.synth.config_data("c2")
    assert m.shape == (int(g["n"]), int(g["d"]))
    final, _ = _run_stepwise("c2", m, g, mti_scan)
    bad = np.flatnonzero(final != g["assignments"].astype(np.int32))
    if bad.size:
        assert near_tie_rows(m, _golden("c2")["prev_means"], bad, EPS_F64).size == bad.size


def test_config3_full_trajectory_matches_reference():
    """c3 at its full n = 66,000,000 (forgy, 50 iterations, MTI)."""
    g = _golden("c3")
    m = kb.synth.config_data("c3")
    assert m.shape == (int(g["n"]), int(g["d"]))
    _run_stepwise("c3", m, g, "auto")
