"""The multi-GPU orchestration over a real NCCL process group (one rank: the box has one
B200, and NCCL refuses two ranks on one device).  The per-iteration exchange goes
through an NCCL all-reduce of a torch CUDA tensor the library writes into, on
torch's stream -- the same calls a world-size-N run makes."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

import paper_1606_08905_b200 as kb
from paper_1606_08905_b200.parallel import TorchComm

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_group():
    import torch
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield TorchComm()
    dist.destroy_process_group()


@pytest.mark.parametrize("init,pruning,f32", [("forgy", True, False), ("kmeanspp", True, False),
                                               ("random-partition", False, False), ("forgy", False, True)])
def test_sharded_over_nccl_equals_single(nccl_group, init, pruning, f32):
    d = 64 if f32 else 12
    m = kb.synth.mixture(kb.synth.MixtureSpec(30000, d, 12, 5, "uniform", -3, 3, 0.8))
    if f32:
        m = m.astype(np.float32)
    cfg = dict(k=12, init=init, seed=3, pruning=pruning, max_iters=15)
    a = kb.kmeans(m, kb.EngineConfig(**cfg))
    # collect_assignments forces the per-iteration loop: local pass -> NCCL all-reduce -> finish
    b = kb.kmeans_sharded(m, kb.EngineConfig(collect_assignments=True, **cfg), nccl_group, n_global=m.shape[0])
    assert a.n_iterations == b.n_iterations
    assert np.array_equal(a.assignments, b.assignments)
    assert np.array_equal(a.centroids.means, b.centroids.means)
    assert [s.wcss for s in a.iterations] == [s.wcss for s in b.iterations]


@pytest.mark.parametrize("init,pruning,f32", [("forgy", True, False), ("kmeanspp", False, False),
                                               ("forgy", False, True)])
def test_sharded_graphed_loop_equals_single(nccl_group, init, pruning, f32):
    """The multi-GPU loop without per-iteration host work: iteration 0 eagerly, then
    replays of one captured iteration (local pass -> NCCL all-reduce -> finish) with the
    stop flag on the device (engine._run_graphed; forced on the one-rank group)."""
    d = 64 if f32 else 12
    m = kb.synth.mixture(kb.synth.MixtureSpec(30000, d, 12, 6, "uniform", -3, 3, 0.8))
    if f32:
        m = m.astype(np.float32)
    cfg = dict(k=12, init=init, seed=4, pruning=pruning, max_iters=40, batch=6)
    a = kb.kmeans(m, kb.EngineConfig(**cfg))
    nccl_group.force_graph = True
    try:
        b = kb.kmeans_sharded(m, kb.EngineConfig(**cfg), nccl_group, n_global=m.shape[0])
    finally:
        nccl_group.force_graph = False
    assert a.n_iterations == b.n_iterations and a.converged == b.converged
    assert np.array_equal(a.assignments, b.assignments)
    assert np.array_equal(a.centroids.means, b.centroids.means)
    assert [s.reassignments for s in a.iterations] == [s.reassignments for s in b.iterations]
