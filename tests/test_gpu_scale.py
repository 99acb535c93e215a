"""Full-scale BASELINE configs on one B200, checked through size-independent
properties (step-wise + sampled parity for configs 4/5)."""

from __future__ import annotations

import numpy as np
import pytest

import paper_1606_08905_b200 as kb
from conftest import EPS_F64, near_tie_rows
from oracle import lloyd as O

pytestmark = pytest.mark.gpu


def test_device_pcg64_is_numpys_stream():
    """default_rng(4).random((n, 16)) bit for bit, from the start and mid-stream."""
    n, d = 200_000, 16
    want = np.random.default_rng(4).random((n, d))
    got = kb.synth.uniform_device(n, d, 4).cpu().numpy()
    assert np.array_equal(got, want)
    for lo, rows in ((1, 7), (31_337, 5000), (n - 3, 3)):
        part = kb.synth.uniform_device(n, d, 4, row_lo=lo, rows=rows).cpu().numpy()
        assert np.array_equal(part, want[lo:lo + rows])


def test_config4_full_size_on_one_gpu():
    """Config 4 at n = 856M (109.6 GB f64 + 11 GB MTI state in one B200's HBM):
    sampled assignments equal the oracle's argmin against the centroids they were made
    with, Sigma counts == n, and the centroids are the f64 means of the GPU's own
    assignment (recomputed independently with torch on the device)."""
    import torch

    n, d, k = 856_000_000, 16, 100
    x = kb.synth.uniform_device(n, d, 4)
    r = kb.kmeans(x, kb.EngineConfig(k=k, init="forgy", seed=4, pruning=True, max_iters=3))
    assert r.n_iterations == 3
    # the forgy rows come from the host RNG stream exactly as the reference draws them
    rows0 = np.sort(np.random.default_rng(4).choice(n, size=k, replace=False))
    assert r.init_rows == [int(i) for i in rows0]
    rng = np.random.default_rng(0)
    sample = np.sort(rng.choice(n, size=4000, replace=False))
    xs = x[torch.from_numpy(sample).cuda()].cpu().numpy()
    ids, _, _ = O.lloyd_step(xs, r.centroids.prev_means)
    bad = np.flatnonzero(ids != r.assignments[sample])
    assert near_tie_rows(xs, r.centroids.prev_means, bad, EPS_F64).size == bad.size
    assert int(r.centroids.counts.sum()) == n
    a = torch.from_numpy(r.assignments.astype(np.int64)).cuda()
    cnt = torch.bincount(a, minlength=k).cpu().numpy()
    assert np.array_equal(cnt, r.centroids.counts)
    sums = torch.zeros((k, d), dtype=torch.float64, device="cuda").index_add_(0, a, x).cpu().numpy()
    means = sums / np.maximum(cnt, 1)[:, None]
    occ = cnt > 0
    assert float(np.abs(means[occ] - r.centroids.means[occ]).max()) < 1e-9
    del x, a
    torch.cuda.empty_cache()
