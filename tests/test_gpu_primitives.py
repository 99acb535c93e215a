"""The reference's public primitives on the GPU (primitives.py) against the pinned
oracle's recipe and the reference tests' own known answers (test_distance.py,
test_pruning.py, test_centroids.py)."""

from __future__ import annotations

import numpy as np
import pytest

import paper_1606_08905_b200 as kb
from oracle import lloyd as O

pytestmark = pytest.mark.gpu


def test_known_answers():
    assert kb.euclidean_distance([0.0, 0.0], [3.0, 4.0]) == 5.0               # test_distance.py:18-19
    ids, best = kb.nearest_centroid(np.array([[0.0]]), np.array([[-1.0], [1.0]]))
    assert ids[0] == 0 and best[0] == 1.0                                    # tie -> lowest id
    g = kb.centroid_geometry(kb.CentroidSet.from_means(np.array([[0.0], [2.0], [6.0]])))
    assert np.array_equal(g.half_dist, np.array([[0, 1, 3], [1, 0, 2], [3, 2, 0]], dtype=float))
    assert np.array_equal(g.half_min, [1.0, 1.0, 2.0])                       # test_pruning.py:36-43
    one = kb.centroid_geometry(kb.CentroidSet.from_means(np.array([[1.0, 2.0]])))
    assert one.half_min[0] == np.inf
    with pytest.raises(ValueError, match="length mismatch"):
        kb.euclidean_distance([1.0, 2.0], [1.0])


@pytest.mark.parametrize("d", [1, 3, 8, 15, 16, 17, 32, 33, 64, 100])
def test_distances_bit_exact_with_the_recipe(d):
    rng = np.random.default_rng(d)
    rows, cents = rng.normal(size=(300, d)) * 3, rng.normal(size=(13, d))
    got = kb.block_distances(rows, cents)
    assert np.array_equal(got, O.dist_matrix(rows, cents))
    ids, best = kb.nearest_centroid(rows, cents)
    want_ids, want_best = O.nearest(rows, cents)
    assert np.array_equal(ids, want_ids) and np.array_equal(best, want_best)
    assert np.array_equal(kb.row_sqnorms(rows), O.sqnorms(rows))
    assert np.array_equal(kb.rowwise_distances(rows, cents[0]), O.dist_to(rows, cents[0]))
    assert np.array_equal(kb.rowwise_distances(rows[:13], cents), np.sqrt(np.vecdot(rows[:13] - cents, rows[:13] - cents)))


@pytest.mark.parametrize("method", ["forgy", "random-partition", "kmeanspp"])
def test_init_centroids_match_reference_init(method):
    m = kb.synth.uniform(700, 5, 31)
    got = kb.init_centroids(m, 6, method, seed=17)
    want = O.init_means(m, 6, method, 17)
    if method == "random-partition":  # group means: the device sums in another order (1e-9 bar)
        assert np.max(np.abs(got.means - want)) <= 1e-12 * np.max(np.abs(want))
    else:                             # gathered rows: identical
        assert np.array_equal(got.means, want)
    given = kb.init_centroids(m, 2, "given", initial=np.ones((2, 5)))
    assert np.array_equal(given.means, np.ones((2, 5)))
    with pytest.raises(ValueError, match="k <= n"):
        kb.init_centroids(m[:3], 6, "forgy")
    with pytest.raises(ValueError, match="unknown init"):
        kb.init_centroids(m, 2, "bogus")
