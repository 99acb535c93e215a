"""GPU parity of the f32 tensor-core path (BASELINE config 5: tcgen05 kind::tf32 scores,
certified argmin, exact f64 rerank of the uncertified rows, cluster-sorted accumulation).

The reference upcasts f32 input to f64 (matrix.py:40) and runs its f64 recipe; the
oracle does the same, so every comparison below is against f64 answers."""

from __future__ import annotations

import numpy as np
import pytest

import paper_1606_08905_b200 as kb
from conftest import EPS_F64, assert_parity, golden, near_tie_rows
from oracle import lloyd as O
from oracle.golden_cases import case_data

pytestmark = pytest.mark.gpu


def _path(m, cfg):
    s = kb.Lloyd(m, cfg)
    try:
        return s.ctx.describe(), s.ctx.tc_info()
    finally:
        s.close()


def test_c5_mini_runs_on_tensor_cores_and_matches_golden():
    g = golden("c5_mini")
    m = case_data("c5_mini")
    assert m.dtype == np.float32
    cfg = dict(k=1000, init="forgy", seed=5, pruning=False, max_iters=g["reassignments"].size)
    desc, info = _path(m, kb.EngineConfig(**cfg))
    assert desc["dense_dp"] < 0 and info["active"], desc
    r = kb.kmeans(m, kb.EngineConfig(collect_assignments=True, **cfg))
    assert_parity(m.astype(np.float64), r, g["means"], g["assignments"], len(g["reassignments"]),
                  want_prev=g["prev_means"], counters={"reassignments": g["reassignments"],
                                                       "dist_comps": g["dist_comps"]},
                  wcss=g["wcss"], what="c5_mini")


@pytest.mark.parametrize("n,d,k,seed", [
    (1000, 32, 5, 0), (3001, 64, 300, 1), (5000, 100, 257, 2), (4097, 128, 1000, 3),
    (2500, 256, 1000, 4), (1777, 256, 1100, 5), (6000, 200, 64, 6), (130, 36, 1, 7)])
def test_tc_matches_oracle(n, d, k, seed):
    """Random f32 mixtures of every shape class the path takes (d not a multiple of 32,
    k not a multiple of 256, n not a multiple of 128, k = 1): assignments every
    iteration, centroids, iteration count, reassignments and WCSS."""
    rng = np.random.default_rng(seed)
    spec = kb.synth.MixtureSpec(n, d, max(1, k // 2), 50 + seed, "normal", 0, 0, 0.3, None, "float32")
    m = kb.synth.mixture(spec)
    if seed % 2:
        m *= np.float32(rng.uniform(0.01, 100.0))
    cfg = dict(k=k, init="forgy", seed=seed, pruning=False, max_iters=6)
    r = kb.kmeans(m, kb.EngineConfig(collect_assignments=True, **cfg))
    o = O.lloyd(m.astype(np.float64), k, init="forgy", seed=seed, pruning=False, max_iters=6, collect=True)
    assert_parity(m.astype(np.float64), r, o.means, o.assignments, o.n_iterations, want_prev=o.prev_means,
                  counters={"reassignments": [s.reassignments for s in o.iterations],
                            "dist_comps": [s.dist_comps for s in o.iterations]},
                  wcss=[s.wcss for s in o.iterations], what=f"tc n={n} d={d} k={k}")
    for a, b in zip(r.assignment_history, o.history):  # every iteration (no near-ties in these draws)
        assert np.array_equal(a, b)


def test_tc_exact_ties_go_to_lowest_id():
    """Duplicated rows picked by forgy give identical centroids: exact score ties, which
    the certificate must send to the exact rerank (lowest id wins, distance.py:114-116)."""
    base = kb.synth.mixture(kb.synth.MixtureSpec(600, 64, 6, 11, "normal", 0, 0, 0.3, None, "float32"))
    m = np.repeat(base, 3, axis=0)  # every row three times
    init = np.stack([m[0], m[1], m[2], m[30], m[31], m[300]]).astype(np.float64)  # rows 0..2 identical
    cfg = dict(k=6, init="given", pruning=False, max_iters=5, initial_centroids=init)
    r = kb.kmeans(m, kb.EngineConfig(collect_assignments=True, **cfg))
    o = O.lloyd(m.astype(np.float64), 6, init="given", initial=init, pruning=False, max_iters=5, collect=True)
    assert r.n_iterations == o.n_iterations
    assert np.array_equal(r.assignment_history[0], o.history[0])
    assert not np.any(r.assignment_history[0] == 1) and not np.any(r.assignment_history[0] == 2)
    assert_parity(m.astype(np.float64), r, o.means, o.assignments, o.n_iterations, want_prev=o.prev_means,
                  wcss=[s.wcss for s in o.iterations], what="ties")
    s = kb.Lloyd(m, kb.EngineConfig(**cfg))
    s.step()
    assert s.ctx.tc_info()["flagged_rows"] >= np.sum(o.history[0] == 0)
    s.close()


def test_tc_device_tensor_and_upcast_paths_agree():
    """f32 CUDA tensor (attached in place), f32 host array (uploaded as f32) and the f64
    upcast (generic exact path) give the same run."""
    import torch
    m = kb.synth.mixture(kb.synth.MixtureSpec(3000, 96, 40, 21, "normal", 0, 0, 0.3, None, "float32"))
    cfg = dict(k=40, init="kmeanspp", seed=2, pruning=False, max_iters=8)
    a = kb.kmeans(m, kb.EngineConfig(**cfg))
    b = kb.kmeans(torch.from_numpy(m).cuda(), kb.EngineConfig(**cfg))
    c = kb.kmeans(m.astype(np.float64), kb.EngineConfig(**cfg))
    assert a.n_iterations == b.n_iterations == c.n_iterations
    assert np.array_equal(a.assignments, b.assignments)
    assert np.array_equal(a.assignments, c.assignments)
    assert np.array_equal(a.centroids.means, b.centroids.means)
    assert np.max(np.abs(a.centroids.means - c.centroids.means)) < 1e-12


def test_tc_random_partition_init_and_repeatability():
    m = kb.synth.mixture(kb.synth.MixtureSpec(5000, 128, 20, 31, "normal", 0, 0, 0.3, None, "float32"))
    cfg = dict(k=20, init="random-partition", seed=4, pruning=False, max_iters=7)
    a = kb.kmeans(m, kb.EngineConfig(**cfg))
    b = kb.kmeans(m, kb.EngineConfig(**cfg))
    assert np.array_equal(a.centroids.means, b.centroids.means)
    assert [s.wcss for s in a.iterations] == [s.wcss for s in b.iterations]
    o = O.lloyd(m.astype(np.float64), 20, init="random-partition", seed=4, pruning=False, max_iters=7)
    assert_parity(m.astype(np.float64), a, o.means, o.assignments, o.n_iterations, want_prev=o.prev_means,
                  wcss=[s.wcss for s in o.iterations], what="random-partition")


def test_tc_config5_sampled_full_size():
    """Config 5 at full size (10M x 256 f32, k = 1000, 3 iterations): sampled rows equal
    the oracle's argmin against the centroids they were assigned with; Sigma counts == n;
    centroids are the f64 means of the GPU's own assignment (torch, on device)."""
    import torch
    n, d, k = 10_000_000, 256, 1000
    g = torch.Generator(device="cuda").manual_seed(5)
    centers = torch.randn((k, d), generator=g, device="cuda", dtype=torch.float32)
    lab = torch.randint(0, k, (n,), generator=g, device="cuda")
    x = centers[lab] + 0.3 * torch.randn((n, d), generator=g, device="cuda", dtype=torch.float32)
    del lab
    r = kb.kmeans(x, kb.EngineConfig(k=k, init="forgy", seed=5, pruning=False, max_iters=3))
    assert r.n_iterations == 3
    rows = np.sort(np.random.default_rng(0).choice(n, size=3000, replace=False))
    xs = x[torch.from_numpy(rows).cuda()].double().cpu().numpy()
    ids, _, _ = O.lloyd_step(xs, r.centroids.prev_means)
    bad = np.flatnonzero(ids != r.assignments[rows])
    assert near_tie_rows(xs, r.centroids.prev_means, bad, EPS_F64).size == bad.size
    a = torch.from_numpy(r.assignments.astype(np.int64)).cuda()
    cnt = torch.bincount(a, minlength=k).cpu().numpy()
    assert np.array_equal(cnt, r.centroids.counts) and cnt.sum() == n
    sums = torch.zeros((k, d), dtype=torch.float64, device="cuda")
    for lo in range(0, n, 1 << 21):
        sums.index_add_(0, a[lo:lo + (1 << 21)], x[lo:lo + (1 << 21)].double())
    means = (sums.cpu().numpy() / np.maximum(cnt, 1)[:, None])
    occ = cnt > 0
    assert float(np.abs(means[occ] - r.centroids.means[occ]).max()) < 1e-9
    del x, a, sums
    torch.cuda.empty_cache()


@pytest.mark.parametrize("law", ["mixture", "positive", "wide"])
def test_tc_score_error_within_half_the_certified_bound(law):
    """The certificate assumes |s~ - s| <= e ||x|| max||c|| (+ rounding terms).  Measure
    the tensor-core scores against f64 on adversarial-ish inputs (all-positive values,
    so no cancellation hides truncation; 24-bit mantissas; mixed magnitudes): the
    largest error must stay under half of e -- a factor-two margin on the model."""
    import torch
    rng = np.random.default_rng({"mixture": 1, "positive": 2, "wide": 3}[law])
    n, d, k = 3000, 256, 600
    if law == "mixture":
        m = kb.synth.mixture(kb.synth.MixtureSpec(n, d, 300, 9, "normal", 0, 0, 0.3, None, "float32"))
    elif law == "positive":
        m = (1.0 + rng.random((n, d))).astype(np.float32)
    else:
        m = (rng.standard_normal((n, d)) * np.exp(rng.uniform(-4, 4, (n, 1)))).astype(np.float32)
    s = kb.Lloyd(m, kb.EngineConfig(k=k, init="forgy", seed=3, pruning=False, max_iters=3))
    s.step()  # centroids become f64 means (not f32-representable)
    kp = (k + 255) // 256 * 256
    out = torch.empty((n, kp), dtype=torch.float32, device="cuda")
    e = s.ctx.tc_scores(out.data_ptr())
    got = out.cpu().numpy()[:, :k].astype(np.float64)
    means, _, _, _ = s.ctx.centroids()
    s.close()
    x = m.astype(np.float64)
    want = x @ means.T - 0.5 * np.einsum("ij,ij->i", means, means)[None, :]
    scale = np.sqrt(np.einsum("ij,ij->i", x, x))[:, None] * np.sqrt(np.max(np.einsum("ij,ij->i", means, means)))
    ratio = float(np.max(np.abs(got - want) / scale))
    assert ratio <= e / 2, (ratio, e)
