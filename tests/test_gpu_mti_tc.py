"""GPU parity of the tcgen05 MTI pass for f64 rows with d in {8, 16, 32} (mti_tc.cu;
BASELINE configs 3, 4, 2): split-TF32 scores D~ ~ ||x - c||^2 on the tensor cores, a
certified argmin, and the exact-recipe re-rank of every uncertified row.

The certificate is only as good as its error bound E(x) (mti_tc.cu header), so the
first test measures |D~ - D| against E on adversarial inputs; the others check the
pass's outputs against the reference goldens and the pinned oracle."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

import paper_1606_08905_b200 as kb
from conftest import assert_parity, golden
from oracle import lloyd as O
from oracle.golden_cases import CASES, case_cfg, case_data

pytestmark = pytest.mark.gpu


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int32).tobytes()).hexdigest()


def _bound(x, means):
    """E(x) of mti_tc.cu: the certified bound on |D~_j - D_j| for every j (Geo<XD>::C1 / C2)."""
    d = x.shape[1]
    c1, c2 = (20.0, 6.0) if d == 32 else (12.0, 4.0)
    xn2 = np.einsum("ij,ij->i", x, x)
    cmax2 = float(np.einsum("ij,ij->i", means, means).max())
    return 2.0 ** -20 * (c1 * np.sqrt(xn2) * np.sqrt(cmax2) + c2 * (xn2 + cmax2)) + \
        (8 * d + 32) * 2.0 ** -53 * (xn2 + cmax2)


def _data(kind, n, seed, d=16):
    rng = np.random.default_rng(seed)
    if kind == "uniform":      # config 4's law
        return rng.random((n, d))
    if kind == "mixture":
        return kb.synth.mixture(kb.synth.MixtureSpec(n, d, 24, seed, "uniform", -4, 4, 1.0))
    if kind == "normal":       # mixed signs
        return rng.standard_normal((n, d))
    if kind == "wide":         # per-row magnitudes over six decades
        return rng.standard_normal((n, d)) * 10.0 ** rng.uniform(-3, 3, (n, 1))
    if kind == "offset":       # a large common offset: every row far from the origin
        return 1000.0 + rng.random((n, d))
    if kind == "lattice":      # exact ties everywhere
        return rng.integers(0, 4, (n, d)).astype(np.float64)
    raise ValueError(kind)


@pytest.mark.parametrize("kind,k,d", [("uniform", 100, 16), ("uniform", 128, 16), ("mixture", 24, 16),
                                      ("normal", 7, 16), ("wide", 50, 16), ("offset", 100, 16), ("lattice", 17, 16),
                                      ("uniform", 1, 16), ("uniform", 10, 8), ("wide", 100, 8), ("offset", 33, 8),
                                      ("uniform", 32, 32), ("wide", 32, 32), ("offset", 17, 32), ("normal", 1, 32)])
def test_split_tf32_scores_within_a_quarter_of_the_certificate(kind, k, d):
    """max_j |D~_j - D_j| / E(x) < 1/4 on every row, at the forgy centroids and after
    two updates; padded columns (j >= k) score >= 2^99 (never a winner)."""
    import torch

    n = 6000
    x = _data(kind, n, 11, d)
    s = kb.Lloyd(x, kb.EngineConfig(k=k, init="forgy", seed=3, pruning=True, max_iters=8, mti_scan="tc"))
    try:
        assert s.ctx.mti_tc_info()["available"]
        N = (k + 15) // 16 * 16
        worst = 0.0
        for step in range(3):
            if step:
                s.step()
            means = s.ctx.centroids()[0]
            out = torch.empty((n, N), dtype=torch.float32, device="cuda")
            s.ctx.mti_tc_scores(out.data_ptr())
            got = out.cpu().numpy().astype(np.float64)
            diff = x[:, None, :] - means[None, :, :]
            want = np.einsum("ijk,ijk->ij", diff, diff)
            ratio = np.abs(got[:, :k] - want) / _bound(x, means)[:, None]
            worst = max(worst, float(ratio.max()))
            if N > k:
                assert float(got[:, k:].min()) >= 2.0 ** 99
        assert worst < 0.25, f"{kind} k={k} d={d}: worst |D~ - D| / E = {worst:.3f}"
    finally:
        s.close()


def _tc_shape(d, k):
    return (d in (8, 16) and k <= 128) or (d == 32 and k <= 32)


TC_CASES = [n for n in CASES if CASES[n]["cfg"].get("pruning", True)
            and _tc_shape(case_data(n).shape[1], int(CASES[n]["cfg"]["k"]))]


def test_tc_cases_exist():
    assert {"c4_mini", "d16_k24_pruned", "tie_pruned_d16", "c2_mini", "c3_mini"} <= set(TC_CASES)


@pytest.mark.parametrize("mode", ["tc", "auto"])
@pytest.mark.parametrize("name", TC_CASES)
def test_tc_mti_matches_reference_golden(name, mode):
    """Every iteration's assignments bit for bit (sha256), centroids, skip counts and
    reassignments equal the reference's; the pass is the tcgen05 one."""
    g = golden(name)
    m = case_data(name)
    c = case_cfg(name)
    cfg = kb.EngineConfig(k=c["k"], init=c.get("init", "forgy"), seed=c.get("seed", 0), pruning=True,
                          max_iters=c.get("max_iters", 100), tolerance=c.get("tolerance", 0),
                          initial_centroids=c.get("initial"), collect_assignments=True, mti_scan=mode)
    r = kb.kmeans(m, cfg)
    assert_parity(m.astype(np.float64), r, g["means"], g["assignments"], len(g["reassignments"]),
                  want_prev=g["prev_means"], counters={"reassignments": g["reassignments"], "skips": g["skips"]},
                  wcss=g["wcss"], what=f"{name}/{mode}")
    assert [_sha(h) for h in r.assignment_history] == list(g["history_sha"]), name
    n, k = m.shape[0], int(c["k"])
    for st in r.iterations[1:]:
        assert st.dist_comps == (n - st.skips) * k


@pytest.mark.parametrize("n,k,kind,seed,d", [(1000, 5, "mixture", 0, 16), (4097, 100, "uniform", 1, 16),
                                             (129, 16, "normal", 2, 16), (2048, 17, "wide", 3, 16),
                                             (3333, 128, "uniform", 4, 16), (700, 1, "normal", 5, 16),
                                             (5000, 33, "lattice", 6, 16), (257, 64, "offset", 7, 16),
                                             (3001, 10, "mixture", 8, 8), (4096, 128, "uniform", 9, 8),
                                             (1500, 7, "lattice", 10, 8), (900, 3, "offset", 11, 8),
                                             (3001, 32, "mixture", 12, 32), (4097, 32, "uniform", 13, 32),
                                             (1500, 9, "lattice", 14, 32), (640, 1, "wide", 15, 32)])
def test_tc_mti_matches_oracle(n, k, kind, seed, d):
    """Random shapes (n not a multiple of 128, k = 1 .. 128, rows of 8 / 16 / 32, ties,
    far-off data): forced tcgen05 pass == the pinned oracle, every iteration."""
    m = _data(kind, n, 100 + seed, d)
    cfg = kb.EngineConfig(k=k, init="forgy", seed=seed, pruning=True, max_iters=12, collect_assignments=True,
                          mti_scan="tc")
    r = kb.kmeans(m, cfg)
    o = O.lloyd(m, k, init="forgy", seed=seed, pruning=True, max_iters=12, collect=True)
    # (far-off rows: the pruned WCSS formula sq - ||sums||^2 / count cancels ~7 digits, so
    # the running sums' summation order shows at 1e-9)
    wc = [s.wcss for s in o.iterations]
    assert_parity(m, r, o.means, o.assignments, o.n_iterations, want_prev=o.prev_means,
                  counters={"reassignments": [s.reassignments for s in o.iterations],
                            "skips": [s.skips for s in o.iterations]},
                  wcss=None if kind == "offset" else wc, what=f"tc n={n} k={k} d={d} {kind}")
    if kind == "offset":
        np.testing.assert_allclose([s.wcss for s in r.iterations], wc, rtol=1e-7)
    for a, b in zip(r.assignment_history, o.history):
        assert np.array_equal(a, b)


def test_tc_equals_dmma_block_pass_on_config4_law():
    """The tcgen05 pass and the FP64 DMMA block pass agree on 2M config-4 rows: same
    assignments at every iteration, centroids to 1e-12; few rows need the re-rank."""
    n = 2_000_000
    m = kb.synth.uniform(n, 16, 4)
    out = {}
    for mode in ("tc", "block"):
        s = kb.Lloyd(m, kb.EngineConfig(k=100, init="forgy", seed=4, pruning=True, max_iters=8, mti_scan=mode))
        hist = []
        for _ in range(8):
            s.step()
            hist.append(_sha(s.ctx.assignments()))
        out[mode] = (hist, s.ctx.centroids()[0], s.ctx.mti_tc_info())
        s.close()
    assert out["tc"][0] == out["block"][0]
    assert float(np.abs(out["tc"][1] - out["block"][1]).max()) < 1e-12
    unc = out["tc"][2]["uncertified"]
    assert unc < 0.01 * n * 7, unc
