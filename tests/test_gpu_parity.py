"""GPU parity: the CUDA path (through the C ABI) against the reference goldens and
the CPU oracle.  Every test here needs a B200 and the built libknorb200.so."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

import paper_1606_08905_b200 as kb
from conftest import EPS_F64, assert_parity, golden, near_tie_rows
from oracle import lloyd as O
from oracle.golden_cases import CASES, case_cfg, case_data

pytestmark = pytest.mark.gpu

COUNTERS = ("reassignments", "dist_comps", "skips", "pruned_stale", "pruned_tight")


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int32).tobytes()).hexdigest()


def _cfg(name, **over):
    c = case_cfg(name)
    kw = dict(k=c["k"], init=c.get("init", "forgy"), seed=c.get("seed", 0), pruning=c.get("pruning", True),
              max_iters=c.get("max_iters", 100), tolerance=c.get("tolerance", 0),
              initial_centroids=c.get("initial"))
    kw.update(over)
    return kb.EngineConfig(**kw)


@pytest.mark.parametrize("name", list(CASES))
def test_gpu_matches_reference_golden(name):
    """mti_scan="exact": every output including the reference's work counters."""
    g = golden(name)
    m = case_data(name)
    r = kb.kmeans(m, _cfg(name, collect_assignments=True, mti_scan="exact"))
    counters = {key: g[key] for key in COUNTERS}
    assert_parity(m.astype(np.float64), r, g["means"], g["assignments"], len(g["reassignments"]),
                  want_prev=g["prev_means"], counters=counters, wcss=g["wcss"], what=name)
    # every iteration's assignment vector, bit for bit
    assert [_sha(h) for h in r.assignment_history] == list(g["history_sha"]), name
    np.testing.assert_array_equal(r.centroids.counts, g["counts"])
    assert r.converged == bool(g["converged"])


@pytest.mark.parametrize("mode", ["auto", "dense", "block"])
@pytest.mark.parametrize("name", [n for n in CASES if CASES[n]["cfg"].get("pruning", True)])
def test_gpu_tensor_core_mti_matches_reference_golden(name, mode):
    """Tensor-core MTI passes (compacted survivors, block-dense, or the device's per-
    iteration choice): assignments every iteration, centroids, bounds-driven skip counts
    and reassignments are the reference's; the distance count is k per survivor."""
    g = golden(name)
    m = case_data(name)
    if m.shape[1] > 64 and mode != "auto":
        pytest.skip("tensor-core MTI needs d <= 64")
    r = kb.kmeans(m, _cfg(name, collect_assignments=True, mti_scan=mode))
    assert_parity(m.astype(np.float64), r, g["means"], g["assignments"], len(g["reassignments"]),
                  want_prev=g["prev_means"], counters={"reassignments": g["reassignments"], "skips": g["skips"]},
                  wcss=g["wcss"], what=name)
    assert [_sha(h) for h in r.assignment_history] == list(g["history_sha"]), name
    n, d, k = m.shape[0], m.shape[1], int(CASES[name]["cfg"]["k"])
    assert r.iterations[0].dist_comps == n * k
    if d <= 64:  # the tensor-core survivor kernel (wider rows keep the exact walk)
        for s in r.iterations[1:]:
            assert s.dist_comps == (n - s.skips) * k
            assert s.pruned_stale == 0 and s.pruned_tight == 0


@pytest.mark.parametrize("name", ["c1_full", "c3_mini", "kpp_pruned", "d33_pruned", "d65_dense", "c5_mini", "unif_pruned"])
def test_gpu_batched_run_equals_stepwise(name):
    """The batched single-GPU loop (CUDA-graph replays, device stop flag) == the
    per-iteration loop."""
    m = case_data(name)
    a = kb.kmeans(m, _cfg(name, batch=7))
    b = kb.kmeans(m, _cfg(name, collect_assignments=True))
    assert a.n_iterations == b.n_iterations
    assert np.array_equal(a.assignments, b.assignments)
    assert np.array_equal(a.centroids.means, b.centroids.means)
    for x, y in zip(a.iterations, b.iterations):
        assert (x.reassignments, x.dist_comps, x.skips, x.wcss) == (y.reassignments, y.dist_comps, y.skips, y.wcss)


def test_repeated_run_bit_identical():
    """test_engine.py:92-101: same config -> identical bits (fixed-order reductions)."""
    m = case_data("k50_pruned")
    a = kb.kmeans(m, _cfg("k50_pruned"))
    b = kb.kmeans(m, _cfg("k50_pruned"))
    assert np.array_equal(a.centroids.means, b.centroids.means)
    assert np.array_equal(a.assignments, b.assignments)
    assert [s.wcss for s in a.iterations] == [s.wcss for s in b.iterations]


def test_validate_bounds_mode():
    """EngineConfig.validate_bounds runs the exhaustive-argmin + bound oracle each iteration."""
    for name in ("mix_pruned", "d17_pruned", "k50_pruned"):
        r = kb.kmeans(case_data(name), _cfg(name, validate_bounds=True, max_iters=12))
        assert r.n_iterations >= 1


@pytest.mark.parametrize("seed", range(6))
def test_pruned_equals_dense_every_iteration(seed):
    """Reference criterion 1 (test_acceptance.py:56-81) on the GPU."""
    rng = np.random.default_rng(900 + seed)
    n = int(rng.integers(1000, 30000))
    d = int(rng.choice([2, 3, 8, 16, 32]))
    k = int(rng.choice([2, 10, 50]))
    m = kb.synth.mixture(kb.synth.MixtureSpec(n, d, 8, 100 + seed, "uniform", -6, 6, 1.0)) \
        if seed % 2 else kb.synth.uniform(n, d, 100 + seed)
    base = dict(k=k, seed=seed + 1, max_iters=8, collect_assignments=True)
    p = kb.kmeans(m, kb.EngineConfig(pruning=True, **base))
    q = kb.kmeans(m, kb.EngineConfig(pruning=False, **base))
    assert p.n_iterations == q.n_iterations
    for a, b in zip(p.assignment_history, q.assignment_history):
        assert np.array_equal(a, b)
    assert np.max(np.abs(p.centroids.means - q.centroids.means)) < 1e-9
    o = O.lloyd(m, k, seed=seed + 1, max_iters=8, pruning=True)
    assert_parity(m, p, o.means, o.assignments, o.n_iterations, want_prev=o.prev_means,
                  counters={key: [getattr(s, key) for s in o.iterations] for key in ("reassignments", "skips")})
    x = kb.kmeans(m, kb.EngineConfig(pruning=True, mti_scan="exact", **base))
    assert_parity(m, x, o.means, o.assignments, o.n_iterations, want_prev=o.prev_means,
                  counters={key: [getattr(s, key) for s in o.iterations] for key in COUNTERS})


def test_large_k_generic_path():
    """k*d too large for shared memory -> generic kernels, same answers."""
    m = kb.synth.uniform(6000, 16, 77)
    cfg = dict(k=2000, seed=3, max_iters=3)
    r = kb.kmeans(m, kb.EngineConfig(pruning=True, mti_scan="exact", **cfg))
    o = O.lloyd(m, 2000, seed=3, max_iters=3, pruning=True)
    assert_parity(m, r, o.means, o.assignments, o.n_iterations, want_prev=o.prev_means,
                  counters={key: [getattr(s, key) for s in o.iterations] for key in COUNTERS})


def test_torch_device_input_is_used_in_place():
    import torch
    m = case_data("kpp_pruned")
    a = kb.kmeans(m, _cfg("kpp_pruned"))
    t = torch.from_numpy(m).cuda()
    b = kb.kmeans(t, _cfg("kpp_pruned"))
    assert np.array_equal(a.assignments, b.assignments)
    assert np.array_equal(a.centroids.means, b.centroids.means)


def test_misaligned_device_view_matches_reference_golden():
    """A CUDA tensor at an 8-byte (not 16-byte) offset: the twelve-warp MTI form needs
    16-byte rows, so the eight-warp form takes over -- same reference results."""
    import torch
    m = case_data("d16_k24_pruned")
    flat = torch.empty(m.size + 1, dtype=torch.float64, device="cuda")
    view = flat[1:].view(m.shape)
    view.copy_(torch.from_numpy(m))
    assert view.data_ptr() % 16 == 8
    r = kb.kmeans(view, _cfg("d16_k24_pruned", collect_assignments=True))
    g = golden("d16_k24_pruned")
    assert r.n_iterations == len(g["reassignments"])
    assert np.array_equal(r.assignments, g["assignments"].astype(np.int32))
    assert np.array_equal([s.skips for s in r.iterations], g["skips"])
    np.testing.assert_allclose(r.centroids.means, g["means"], rtol=0, atol=1e-9 * np.abs(g["means"]).max())


def test_nonfinite_rejected_on_device():
    m = kb.synth.uniform(5000, 4, 1)
    m[3210, 2] = np.inf
    with pytest.raises(kb.MatrixFormatError, match="row 3210"):
        kb.kmeans(m, kb.EngineConfig(k=3))


def test_forgy_k_gt_n_message():
    with pytest.raises(ValueError, match="k <= n"):
        kb.kmeans(np.random.default_rng(0).normal(size=(10, 2)), kb.EngineConfig(k=11, init="forgy"))


def test_k1_and_more_workers_than_rows():
    m = np.random.default_rng(1234).normal(size=(100, 3))
    r = kb.kmeans(m, kb.EngineConfig(k=1, pruning=False))
    assert r.n_iterations == 1 and r.converged
    assert np.allclose(r.centroids.means[0], m.mean(axis=0))
    m3 = np.random.default_rng(5).normal(size=(3, 2))
    for pruning in (False, True):
        r = kb.kmeans(m3, kb.EngineConfig(k=2, seed=1, T=8, pruning=pruning, max_iters=10))
        assert r.converged and int(r.centroids.counts.sum()) == 3


def test_wcss_non_increasing_and_counts():
    for name in ("unif_dense", "unif_pruned", "mix_pruned", "c3_mini"):
        r = kb.kmeans(case_data(name), _cfg(name))
        w = [s.wcss for s in r.iterations]
        assert all(b <= a * (1 + 1e-9) for a, b in zip(w, w[1:])), name
        assert int(r.centroids.counts.sum()) == case_data(name).shape[0]


def test_lloyd_step_api_matches_kmeans():
    m = case_data("c4_mini")
    cfg = _cfg("c4_mini", max_iters=6)
    full = kb.kmeans(m, cfg)
    s = kb.Lloyd(m, _cfg("c4_mini", max_iters=6))
    for _ in range(6):
        s.step()
    s.sync()
    means, _, _, _ = s.ctx.centroids()
    assert np.array_equal(s.ctx.assignments(), full.assignments)
    assert np.array_equal(means, full.centroids.means)
    s.close()


def _stepwise_sample_check(m, r, sample=20000, seed=0):
    """Size-independent properties at full scale: sampled assignments equal the oracle's
    argmin against the centroids they were made with (near-ties excepted); centroids are
    the f64 means of the GPU's own assignment; Sigma counts == n."""
    n, d = m.shape
    rng = np.random.default_rng(seed)
    rows = np.sort(rng.choice(n, size=min(sample, n), replace=False))
    ids, _, _ = O.lloyd_step(m[rows], r.centroids.prev_means)
    bad = rows[ids != r.assignments[rows]]
    assert near_tie_rows(m, r.centroids.prev_means, bad, EPS_F64).size == bad.size
    k = r.centroids.k
    counts = np.bincount(r.assignments, minlength=k)
    assert np.array_equal(counts, r.centroids.counts)
    assert counts.sum() == n
    sums = np.stack([np.bincount(r.assignments, weights=m[:, e], minlength=k) for e in range(d)], axis=1)
    occ = counts > 0
    want = r.centroids.means.copy()
    want[occ] = sums[occ] / counts[occ, None]
    scale = max(1.0, float(np.abs(want).max()))
    assert float(np.abs(want - r.centroids.means).max()) / scale < 1e-9


def test_config3_full_size_properties():
    """Config 3 at its full n = 66M (4.2 GB): pruned == dense assignments after 6
    iterations, sampled oracle argmin, exact means of the GPU's own assignment."""
    cfg = kb.synth.CONFIGS["c3"]
    m = cfg["data"](cfg["n"])
    p = kb.kmeans(m, kb.EngineConfig(k=10, init="forgy", seed=3, pruning=True, max_iters=6))
    q = kb.kmeans(m, kb.EngineConfig(k=10, init="forgy", seed=3, pruning=False, max_iters=6))
    assert p.n_iterations == q.n_iterations == 6
    assert np.array_equal(p.assignments, q.assignments)
    assert [s.reassignments for s in p.iterations] == [s.reassignments for s in q.iterations]
    _stepwise_sample_check(m, p)


def test_config4_shape_sample():
    """Config 4's law (U[0,1)^16, k=100) at 8M rows (1 GB): stepwise sampled parity."""
    m = kb.synth.uniform(8_000_000, 16, 4)
    r = kb.kmeans(m, kb.EngineConfig(k=100, init="forgy", seed=4, pruning=True, max_iters=3))
    assert r.n_iterations == 3
    _stepwise_sample_check(m, r, sample=5000)


@pytest.mark.parametrize("n,d,k,seed", [(5000, 5, 20, 1), (20000, 32, 32, 2), (3000, 100, 12, 3), (4000, 3, 50, 4)])
def test_gpu_kmeanspp_device_loop_matches_oracle(n, d, k, seed):
    """The single-GPU kmeans++ loop (knb_kpp_run: every D^2 update, total and search on
    the device) picks exactly the reference's rows (oracle pinned to the reference)."""
    m = kb.synth.mixture(kb.synth.MixtureSpec(n, d, max(2, k // 2), 40 + seed, "uniform", -4, 4, 1.0))
    r = kb.kmeans(m, kb.EngineConfig(k=k, init="kmeanspp", seed=seed, pruning=True, max_iters=2))
    o = O.lloyd(m, k, init="kmeanspp", seed=seed, pruning=True, max_iters=2)
    np.testing.assert_array_equal(m[np.asarray(r.init_rows)], o.init_means)


def test_gpu_kmeanspp_degenerate_total_replays_reference_draws():
    """Only two distinct points and k = 3: after both are picked every D^2 is 0 and the
    reference draws rng.integers(n) instead of a weighted choice (centroids.py:182-186);
    the device loop reports it and the host replays the reference's draw order."""
    m = np.array([[0.0, 0.0]] * 3 + [[1.0, 1.0]] * 2)
    for seed in range(6):
        r = kb.kmeans(m, kb.EngineConfig(k=3, init="kmeanspp", seed=seed, pruning=False, max_iters=3))
        o = O.lloyd(m, 3, init="kmeanspp", seed=seed, pruning=False, max_iters=3)
        np.testing.assert_array_equal(m[np.asarray(r.init_rows)], o.init_means)
        assert np.array_equal(r.centroids.means, o.means)


@pytest.mark.parametrize("name", ["kpp_prune", "forgy_dense", "rp_prune_tol", "sem_cache", "sem_nocache_pages",
                                  "sem_plain"])
def test_gpu_cli_train_report_matches_reference_report(name, tmp_path):
    """The command line (``train`` on a KNRM file the reference wrote) reproduces the
    reference CLI's report: every counter of every iteration, the totals and the
    convergence line exactly (mti_scan="exact" keeps the reference's clause-2/3
    counters), the WCSS column to 1e-9; ``--mode sem`` runs add the reference's I/O
    columns (bytes requested / read, cache hits / misses, rows elided), also exact."""
    import os
    from paper_1606_08905_b200.cli import main
    from paper_1606_08905_b200.report import TIMING_FIELDS, parse_report
    gold = os.path.join(os.path.dirname(__file__), "golden", "reports")
    with open(os.path.join(gold, f"{name}.args")) as fh:
        argv = fh.read().split()
    out = tmp_path / "r.txt"
    cwd = os.getcwd()
    os.chdir(os.path.dirname(os.path.dirname(__file__)))
    try:
        assert main(["train", "--data", f"tests/golden/reports/{name}.knrm", *argv, "--mti-scan", "exact",
                     "--report", str(out)]) == 0
    finally:
        os.chdir(cwd)
    ours = parse_report(out.read_text())
    with open(os.path.join(gold, f"{name}.report")) as fh:
        ref = parse_report(fh.read())
    assert ours["config"] == ref["config"] and ours["converged"] == ref["converged"]
    assert len(ours["iterations"]) == len(ref["iterations"])
    for a, b in zip(ours["iterations"], ref["iterations"]):
        for key in a:
            if key in TIMING_FIELDS:
                continue
            if key == "wcss":
                assert abs(a[key] - b[key]) <= 1e-9 * abs(b[key]), (key, a, b)
            else:
                assert a[key] == b[key], (key, a, b)
    assert {k: v for k, v in ours["totals"].items() if k not in TIMING_FIELDS} == \
        {k: v for k, v in ref["totals"].items() if k not in TIMING_FIELDS}


@pytest.mark.parametrize("pruning", [True, False])
def test_gpu_host_rows_equal_hbm_rows(pruning, tmp_path):
    """Rows left in host memory (page-locked, read over the link; here a memory-mapped
    KNRM file): identical results to the HBM copy, and per-iteration link traffic with
    the clause-1 skipped rows elided."""
    from paper_1606_08905_b200.fileio import load_matrix, save_matrix
    m = kb.synth.mixture(kb.synth.MixtureSpec(40000, 12, 16, 9, "uniform", -5, 5, 0.7))
    path = tmp_path / "x.knrm"
    save_matrix(m, path)
    cfg = dict(k=16, init="kmeanspp", seed=9, pruning=pruning, max_iters=12)
    a = kb.kmeans(m, kb.EngineConfig(**cfg))
    b = kb.kmeans(load_matrix(path, check_finite=False), kb.EngineConfig(host_rows=True, **cfg))
    assert a.n_iterations == b.n_iterations
    assert np.array_equal(a.assignments, b.assignments)
    assert np.array_equal(a.centroids.means, b.centroids.means)
    row = 12 * 8
    assert b.iterations[0].io.bytes_read == 40000 * row
    for s in b.iterations:
        assert s.io.rows_elided == s.skips
        assert s.io.bytes_read == (s.dist_comps // 16) * row
    if pruning:
        assert b.io_totals.rows_elided > 0
        assert b.io_totals.bytes_read < b.n_iterations * 40000 * row


def test_gpu_host_rows_plain_array():
    m = kb.synth.uniform(30000, 8, 5)
    cfg = dict(k=7, init="forgy", seed=5, pruning=True, max_iters=8)
    a = kb.kmeans(m, kb.EngineConfig(**cfg))
    b = kb.kmeans(m, kb.EngineConfig(host_rows=True, **cfg))
    assert np.array_equal(a.assignments, b.assignments)
    assert np.array_equal(a.centroids.means, b.centroids.means)
    assert b.io_totals is not None and a.io_totals is None


def test_gpu_device_mismatch_is_rejected():
    """A CUDA tensor on one device with EngineConfig.device naming another."""
    import torch
    x = torch.zeros((8, 2), dtype=torch.float64, device="cuda:0")
    with pytest.raises(ValueError, match="device"):
        kb.kmeans(x, kb.EngineConfig(k=2, device=1))


@pytest.mark.parametrize("pruning", [False, True])
def test_gpu_large_common_offset_matches_oracle(pruning):
    """Rows around 1e8 with unit spread: the plain engine's running sums move by signed
    deltas after the first pass (the reference recomputes them, engine.py:376-377); the
    centroids stay within the parity bar of the oracle's over many iterations."""
    rng = np.random.default_rng(17)
    centers = 1e8 + rng.uniform(-20, 20, (6, 5))
    m = centers[rng.integers(0, 6, 20000)] + rng.standard_normal((20000, 5))
    cfg = dict(k=6, init="forgy", seed=3, pruning=pruning, max_iters=40)
    r = kb.kmeans(m, kb.EngineConfig(collect_assignments=True, **cfg))
    o = O.lloyd(m, 6, init="forgy", seed=3, pruning=pruning, max_iters=40, collect=True)
    assert_parity(m, r, o.means, o.assignments, o.n_iterations, want_prev=o.prev_means,
                  counters={"reassignments": [s.reassignments for s in o.iterations]},
                  what=f"offset pruning={pruning}")
    # and in units of the spread, not of the 1e8 offset
    assert float(np.abs(r.centroids.means - o.means).max()) < 1e-6


@pytest.mark.parametrize("mode", ["auto", "dense", "block", "exact"])
def test_skewed_row_order_matches_oracle(mode):
    """SURVEY 8(f) f4 / reference test_engine.py:71-89 (results do not depend on the
    scheduling policy): rows sorted by their first-pass cluster, so the clause-1 survivors
    arrive in long contiguous runs and whole row ranges are skipped.  The compacted MTI
    pass deals 32-row blocks round-robin over the grid; every output equals the oracle's
    on the same (sorted) rows, and the assignments are the generated-order run's permuted."""
    m = kb.synth.mixture(kb.synth.MixtureSpec(60_000, 16, 20, 31, "uniform", -5, 5, 0.6, 1.0))
    first = O.lloyd(m, 20, init="forgy", seed=3, pruning=True, max_iters=1)
    order = np.argsort(first.assignments, kind="stable")
    ms = np.ascontiguousarray(m[order])
    init = first.prev_means
    cfg = kb.EngineConfig(k=20, init="given", initial_centroids=init, pruning=True, max_iters=30, mti_scan=mode)
    got = kb.kmeans(ms, cfg)
    want = O.lloyd(ms, 20, init="given", initial=init, pruning=True, max_iters=30)
    assert got.n_iterations == want.n_iterations
    assert np.array_equal(got.assignments, want.assignments)
    for a, b in zip(got.iterations, want.iterations):
        assert (a.reassignments, a.skips) == (b.reassignments, b.skips)
    assert max(s.skips for s in got.iterations) > 0.25 * ms.shape[0]  # long skipped runs did occur
    plain = kb.kmeans(m, cfg)
    assert np.array_equal(plain.assignments[order], got.assignments)


def test_validate_bounds_catches_a_stale_row():
    """The validator's negative case (engine.py:428-445 raises on either violation): after a
    few pruned iterations on well-separated clusters, a row that clause 1 keeps skipping is
    overwritten IN PLACE (the rows are attached device memory) with another cluster's
    centroid.  The next local pass skips it again, so its stored assignment is no longer the
    argmin and its bound is below its true distance -- knb_validate must report that row for
    both checks, and kmeans(validate_bounds=True) semantics (an AssertionError) follow."""
    import torch

    m = kb.synth.mixture(kb.synth.MixtureSpec(20_000, 8, 6, 17, "uniform", -20, 20, 0.05, 1.0))
    x = torch.from_numpy(m).cuda()
    cfg = kb.EngineConfig(k=6, init="kmeanspp", seed=5, pruning=True, max_iters=40, validate_bounds=True)
    run = kb.Lloyd(x, cfg, ignore_stop=True)
    try:
        for _ in range(6):
            run.step()
        run.local()
        run.exchange()
        assert run.ctx.validate() == (-1, -1)
        run.finish()
        means = run.ctx.centroids()[0]
        a = run.ctx.assignments()
        row = 4321
        other = (int(a[row]) + 1) % 6
        assert np.linalg.norm(means[other] - means[a[row]]) > 5.0  # separated clusters
        x[row] = torch.from_numpy(means[other]).cuda()
        torch.cuda.synchronize()
        run.local()  # clause 1 skips the row (its bound still says "close to its centroid")
        run.exchange()
        bad_assign, bad_bound = run.ctx.validate()
        assert bad_assign == row and bad_bound == row, (bad_assign, bad_bound)
    finally:
        run.close()


@pytest.mark.parametrize("mode", ["auto", "dense", "block", "exact"])
def test_sqrt_collision_keeps_the_current_centroid(mode):
    """scan_block compares sqrt'ed distances (pruning.py:190-203).  Here the survivor (0, 0)
    has squared distances 1 + 2^-52 to its own centroid and exactly 1 to another one: the
    square roots collide at 1.0, so the reference keeps the current centroid (a scan on the
    squared values would move the row).  The centroids are fixed points of the update, the
    third one keeps clause 1 from skipping the row; the direct-scan kernel (rows of <= 8
    doubles, k <= 16) must take its sqrt-domain path."""
    e = 2.0 ** -26
    x = np.array([[0, 0], [2, 2 * e]] + [[-1, 0]] * 4 + [[1, 1.5]] * 4, dtype=np.float64)
    init = np.array([[1, e], [-1, 0], [1, 1.5]])
    d0 = x[0] - init[0]
    assert float(d0 @ d0) > 1.0 and float(np.sqrt(d0 @ d0)) == 1.0
    want = O.lloyd(x, 3, init="given", initial=init, pruning=True, max_iters=10)
    assert want.n_iterations == 2 and list(want.assignments[:2]) == [0, 0]
    got = kb.kmeans(x, kb.EngineConfig(k=3, init="given", initial_centroids=init, pruning=True, max_iters=10,
                                       mti_scan=mode))
    assert got.n_iterations == want.n_iterations
    assert np.array_equal(got.assignments, want.assignments)
    for a, b in zip(got.iterations, want.iterations):
        assert (a.reassignments, a.skips) == (b.reassignments, b.skips)


@pytest.mark.parametrize("seed", range(10))
def test_direct_scan_shapes_match_oracle(seed):
    """Rows of <= 8 doubles with k <= 16 (the direct exact-recipe scan of the dense and the
    compacted MTI kernels) on random shapes against the oracle: mixtures, and integer
    lattices whose exact ties exercise scan_block's keep-the-current-centroid rule and the
    full pass's lowest-id rule (pruning.py:174-203, distance.py:106-116)."""
    rng = np.random.default_rng(4100 + seed)
    n = int(rng.integers(200, 12000))
    d = int(rng.integers(1, 9))
    k = int(rng.integers(1, 17))
    if seed % 2:
        m = rng.integers(-3, 4, size=(n, d)).astype(np.float64)  # lattice: many exact ties
    else:
        m = kb.synth.mixture(kb.synth.MixtureSpec(n, d, max(2, k // 2), 77 + seed, "uniform", -4, 4, 0.8, 1.0))
    pruning = seed % 3 != 2
    for mode in (("auto", "dense", "block") if pruning else ("auto",)):
        got = kb.kmeans(m, kb.EngineConfig(k=k, init="forgy", seed=seed, pruning=pruning, max_iters=15,
                                           mti_scan=mode))
        want = O.lloyd(m, k, init="forgy", seed=seed, pruning=pruning, max_iters=15)
        assert got.n_iterations == want.n_iterations, (n, d, k, mode)
        assert np.array_equal(got.assignments, want.assignments), (n, d, k, mode)
        for a, b in zip(got.iterations, want.iterations):
            assert (a.reassignments, a.skips) == (b.reassignments, b.skips), (n, d, k, mode)
        np.testing.assert_allclose(got.centroids.means, want.means, rtol=1e-9, atol=1e-12)
