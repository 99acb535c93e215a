"""Host-side logic and API contract of the drop-in (CPU only)."""

from __future__ import annotations

import numpy as np
import pytest

import paper_1606_08905_b200 as kb
from paper_1606_08905_b200.centroids import check_init
from paper_1606_08905_b200.parallel import group_labels, pick_owner, shard_of


def test_public_names_mirror_reference():
    for name in ("kmeans", "EngineConfig", "KmeansResult", "IterationStats", "CentroidSet",
                 "partition_rows", "check_matrix", "MatrixFormatError", "IoDelta"):
        assert hasattr(kb, name)
    cfg = kb.EngineConfig(k=3)
    # reference defaults (engine.py:59-76)
    assert (cfg.max_iters, cfg.init, cfg.seed, cfg.T, cfg.N, cfg.task_size, cfg.pruning, cfg.mode,
            cfg.tolerance, cfg.scheduler, cfg.collect_assignments, cfg.validate_bounds) == \
        (100, "forgy", 0, 1, 0, 8192, True, "im", 0, "numa", False, False)


@pytest.mark.parametrize("kw", [dict(k=0), dict(k=2, max_iters=0), dict(k=2, task_size=0), dict(k=2, T=0),
                                dict(k=2, N=-1), dict(k=2, tolerance=-1), dict(k=2, init="bogus"),
                                dict(k=2, scheduler="bogus")])
def test_config_validation_errors(kw):
    """test_engine.py:166-180: raised before any device work."""
    with pytest.raises(ValueError):
        kb.kmeans(np.zeros((10, 2)), kb.EngineConfig(**kw))


def test_sem_mode_rejected():
    with pytest.raises(ValueError, match="in-memory"):
        kb.kmeans(np.zeros((10, 2)), kb.EngineConfig(k=2, mode="sem"))


def test_matrix_checks():
    with pytest.raises(kb.MatrixFormatError):
        kb.kmeans(np.zeros(5), kb.EngineConfig(k=1))
    with pytest.raises(kb.MatrixFormatError):
        kb.kmeans(np.zeros((0, 3)), kb.EngineConfig(k=1))
    m = np.zeros((4, 2))
    m[2, 1] = np.nan
    with pytest.raises(kb.MatrixFormatError, match="row 2"):
        kb.check_matrix(m)


def test_init_argument_errors_match_reference_messages():
    with pytest.raises(ValueError, match="k <= n"):
        check_init("forgy", 11, 10, 2, None)
    with pytest.raises(ValueError, match="k <= n"):
        check_init("kmeanspp", 5, 4, 2, None)
    with pytest.raises(ValueError):
        check_init("given", 2, 4, 2, np.ones((3, 2)))
    with pytest.raises(ValueError):
        check_init("given", 2, 4, 2, np.array([[np.inf, 0], [0, 0]]))
    with pytest.raises(ValueError):
        check_init("given", 2, 4, 2, None)


@pytest.mark.parametrize("n,parts", [(10, 3), (3, 8), (1000, 7), (0, 2), (856_000_000, 8)])
def test_partition_rows_matches_reference_rule(n, parts):
    rr = kb.partition_rows(n, parts)
    assert rr[0].start == 0 and rr[-1].stop == n
    sizes = [len(r) for r in rr]
    assert max(sizes) - min(sizes) <= 1
    assert sizes == sorted(sizes, reverse=True)  # remainder to the low ids
    for w, r in enumerate(rr):
        assert shard_of(n, w, parts) == (r.start, r.stop)


@pytest.mark.parametrize("n,k", [(10, 3), (3001, 7), (5, 8), (100, 1)])
def test_group_labels_equal_array_split(n, k):
    perm = np.random.default_rng(n + k).permutation(n)
    labels = group_labels(n, k, perm)
    for j, g in enumerate(np.array_split(perm, k)):
        assert (labels[g] == j).all()


def test_pick_owner():
    assert pick_owner([0.5, 0.5], 0.2) == (0, 0.2)
    r, t = pick_owner([0.5, 0.5], 0.7)
    assert r == 1 and abs(t - 0.2) < 1e-15
    assert pick_owner([0.0, 1.0], 0.1) == (1, 0.1)
    # rounding past the end goes to the last rank holding mass
    assert pick_owner([0.3, 0.7, 0.0], 1.0 + 1e-15)[0] == 1


def test_float32_input_routing():
    """float32 rows stay float32 only where the tcgen05 path serves the configuration
    (dense, 32 <= d <= 256, d % 4 == 0); everything else is upcast like check_matrix."""
    from paper_1606_08905_b200.engine import _rows_of
    m32 = np.ones((10, 64), dtype=np.float32)
    host, dev = _rows_of(m32, kb.EngineConfig(k=3, pruning=False))
    assert dev is None and host.dtype == np.float32 and host.flags.c_contiguous
    host, _ = _rows_of(m32, kb.EngineConfig(k=3, pruning=True))
    assert host.dtype == np.float64
    host, _ = _rows_of(np.ones((10, 6), dtype=np.float32), kb.EngineConfig(k=3, pruning=False))
    assert host.dtype == np.float64
    host, _ = _rows_of(np.ones((10, 64)), kb.EngineConfig(k=3, pruning=False))
    assert host.dtype == np.float64
    with pytest.raises(kb.MatrixFormatError):
        _rows_of(np.ones((0, 64), dtype=np.float32), kb.EngineConfig(k=3, pruning=False))


def test_engine_config_scan_option_validated():
    kb.EngineConfig(k=2, mti_scan="exact").validate()
    with pytest.raises(ValueError, match="mti_scan"):
        kb.EngineConfig(k=2, mti_scan="fast").validate()
