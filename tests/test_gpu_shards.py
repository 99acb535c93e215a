"""Row-sharded runs on the real kernels (multi-GPU readiness): two or three
shards of one matrix, each a context of its own with row_lo > 0 for all but the first,
driven through ``kmeans_sharded`` by threads of one process on the single test GPU
(tests/thread_comm.py: the exchange vectors are summed in rank order between the local
pass and the finish; kmeans++ / forgy / random-partition run their cross-shard
collectives).  Results must equal the single-process reference goldens (assignments of
every shard at every iteration, centroids, counters), as the gloo tests check for the
host orchestration with an oracle-backed shard."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

import paper_1606_08905_b200 as kb
from conftest import assert_parity, golden
from oracle.golden_cases import case_cfg, case_data
from thread_comm import run_ranks

pytestmark = pytest.mark.gpu


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int32).tobytes()).hexdigest()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name", ["mix_pruned", "kpp_pruned", "rp_dense", "d16_k24_pruned", "c4_mini", "c5_mini",
                                  "tie_pruned_d16"])
def test_sharded_kernels_match_reference_golden(name, world):
    g = golden(name)
    m = case_data(name)
    c = case_cfg(name)
    n = m.shape[0]
    if n < 2 * world:
        pytest.skip("too few rows to shard")

    def rank(r, comm):
        lo, hi = kb.shard_of(n, r, world)
        cfg = kb.EngineConfig(k=c["k"], init=c.get("init", "forgy"), seed=c.get("seed", 0),
                              pruning=c.get("pruning", True), max_iters=c.get("max_iters", 100),
                              tolerance=c.get("tolerance", 0), initial_centroids=c.get("initial"),
                              collect_assignments=True, device=0)
        return kb.kmeans_sharded(m[lo:hi], cfg, comm, n_global=n, device=0)

    res = run_ranks(world, rank)
    assert [r.row_lo for r in res] == [kb.shard_of(n, r, world)[0] for r in range(world)]
    full = np.concatenate([r.assignments for r in res])
    hist = [np.concatenate([r.assignment_history[t] for r in res]) for t in range(res[0].n_iterations)]

    class Whole:  # the sharded run seen as one result
        assignments = full
        centroids = res[0].centroids
        iterations = res[0].iterations
        n_iterations = res[0].n_iterations

    assert_parity(m.astype(np.float64), Whole, g["means"], g["assignments"], len(g["reassignments"]),
                  want_prev=g["prev_means"], counters={"reassignments": g["reassignments"], "skips": g["skips"]},
                  wcss=g["wcss"], what=f"{name} x{world}")
    assert [_sha(h) for h in hist] == list(g["history_sha"]), name
    for r in res[1:]:  # every rank finalizes the same centroids
        assert np.array_equal(r.centroids.means, res[0].centroids.means)
