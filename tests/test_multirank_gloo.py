"""World-size-2 coverage of the multi-GPU host path on CPU (gloo).

Each rank hands ``kmeans_sharded`` its contiguous shard (the partition_rows
split); the product's orchestration shards the rows, all-reduces the exchange
vector once per iteration, samples kmeans++ across ranks, gathers forgy rows
from their owners and slices random-partition labels.  The per-shard compute
is the oracle-backed ``FakeContext`` (tests only), so the result must equal
the single-process reference golden.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, out_dir, overrides):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist

    import paper_1606_08905_b200 as kb
    from fake_shard import FakeContext
    from oracle.golden_cases import case_cfg, case_data

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = case_data(name).astype(np.float64)
        c = case_cfg(name)
        c.update(overrides)
        lo, hi = kb.shard_of(m.shape[0], rank, world)
        cfg = kb.EngineConfig(k=c["k"], init=c.get("init", "forgy"), seed=c.get("seed", 0),
                              pruning=c.get("pruning", True), max_iters=c.get("max_iters", 100),
                              tolerance=c.get("tolerance", 0), initial_centroids=c.get("initial"),
                              collect_assignments=True, validate_bounds=c.get("validate", False))
        r = kb.kmeans_sharded(m[lo:hi], cfg, kb.TorchComm(), n_global=m.shape[0], context_cls=FakeContext)
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), assign=r.assignments, means=r.centroids.means,
                 counts=r.centroids.counts, iters=r.n_iterations, row_lo=r.row_lo,
                 reassign=[s.reassignments for s in r.iterations],
                 comps=[s.dist_comps for s in r.iterations], skips=[s.skips for s in r.iterations],
                 init_rows=np.array(r.init_rows if r.init_rows is not None else [], dtype=np.int64))
    finally:
        dist.destroy_process_group()


def _spawn(name, tmp_path, world=2, **overrides):
    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(world, _free_port(), name, str(tmp_path), overrides), nprocs=world, join=True)
    return [np.load(os.path.join(tmp_path, f"r{r}.npz")) for r in range(world)]


@pytest.mark.parametrize("name", ["mix_pruned", "kpp_pruned", "rp_dense", "unif_dense", "d17_pruned"])
def test_two_ranks_match_single_process_reference(name, tmp_path):
    from conftest import golden
    g = golden(name)
    parts = _spawn(name, tmp_path)
    assign = np.concatenate([p["assign"] for p in parts])
    assert all(int(p["iters"]) == len(g["reassignments"]) for p in parts)
    assert np.array_equal(assign, g["assignments"].astype(np.int32))
    for p in parts:
        assert np.array_equal(p["reassign"], g["reassignments"])
        assert np.array_equal(p["comps"], g["dist_comps"])
        assert np.array_equal(p["skips"], g["skips"])
        assert np.array_equal(p["counts"], g["counts"])
        scale = max(1.0, float(np.abs(g["means"]).max()))
        assert float(np.abs(p["means"] - g["means"]).max()) / scale < 1e-9
    # ranks hold identical centroids (redundant finalize on all-reduced inputs)
    assert np.array_equal(parts[0]["means"], parts[1]["means"])
    assert [int(p["row_lo"]) for p in parts] == [0, int(parts[0]["assign"].shape[0])]


def test_three_ranks_kmeanspp_picks_equal_single_process(tmp_path):
    """kmeans++ sampling across 3 shards consumes the RNG stream exactly like one process."""
    from oracle import lloyd as O
    from oracle.golden_cases import case_data
    parts = _spawn("kpp_pruned", tmp_path, world=3, max_iters=2)
    want = O.kmeanspp_picks(case_data("kpp_pruned"), 8, 9)
    for p in parts:
        assert p["init_rows"].tolist() == want


def test_validate_bounds_across_ranks(tmp_path):
    parts = _spawn("mix_pruned", tmp_path, validate=True)
    assert all(int(p["iters"]) >= 1 for p in parts)
