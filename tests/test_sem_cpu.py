"""§8(f) f2 on CPU: the semi-external I/O oracle pinned against the reference's own
kmeans_ondisk runs (tests/golden/sem/, made by oracle/make_golden_sem.py), and the
host side of the out-of-core API (RowStore, page_runs, fetch_rows, the refresh
schedule) on the reference's test_sem.py cases."""

from __future__ import annotations

import hashlib
import os

import numpy as np
import pytest

import paper_1606_08905_b200 as kb
from conftest import ROOT
from oracle import lloyd as O
from oracle import outofcore as OC
from oracle.golden_cases import SEM_CASES, sem_case
from paper_1606_08905_b200.outofcore import (CacheSchedule, IoStats, RowStore, fetch_rows, kmeans_ondisk,
                                             page_runs, rows_per_partition, should_refresh)

SEM_GOLD = os.path.join(ROOT, "tests", "golden", "sem")


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int32).tobytes()).hexdigest()


def sem_oracle(name):
    """(oracle run, io counters, published cache ids) for a golden SEM case."""
    m, cfg, io, page, start = sem_case(name)
    n, d = m.shape
    T, ts = cfg.get("T", 1), cfg.get("task_size", 8192)
    o = O.lloyd(m, cfg["k"], init=cfg.get("init", "forgy"), seed=cfg["seed"], pruning=cfg.get("pruning", True),
                max_iters=cfg["max_iters"], T=T, task_size=ts, collect=True, collect_fetch=True)
    enabled, cap = io.get("cache_enabled", True), io.get("cache_capacity", 64 << 20)
    cnt = OC.io_counters(o.fetched, [s.skips for s in o.iterations], n, d, T, ts, page, enabled, cap, start)
    ids = OC.cached_ids(o.fetched, n, d, T, cap, start) if enabled else np.zeros(0, np.int64)
    return o, cnt, ids


@pytest.mark.parametrize("name", list(SEM_CASES))
def test_sem_oracle_matches_reference_golden(name):
    g = np.load(os.path.join(SEM_GOLD, f"{name}.npz"))
    o, cnt, ids = sem_oracle(name)
    assert [_sha(h) for h in o.history] == list(g["history_sha"])
    assert np.array_equal(cnt, g["io"])
    assert np.array_equal(np.sort(ids), g["cached_ids"])
    assert np.array_equal(o.means, g["means"])


def test_pages_of_equals_page_runs():
    rng = np.random.default_rng(0)
    for rb, ps in ((64, 4096), (24, 512), (2400, 4096), (8, 1000), (4096, 4096), (5000, 4096)):
        ids = np.sort(rng.choice(5000, size=300, replace=False))
        assert OC.pages_of(ids, rb, ps) == page_runs(ids, rb, ps)[1]


@pytest.fixture
def store_8(tmp_path):
    m = kb.synth.uniform(512, 8, 5)  # 64-byte rows, payload exactly 8 pages
    path = tmp_path / "m.raw"
    m.tofile(path)
    with RowStore(path, 512, 8) as store:
        yield store, m


def test_page_accounting(tmp_path, store_8):
    store, m = store_8
    stats = IoStats()
    rows = fetch_rows(store, np.array([0]), None, stats)
    assert (stats.bytes_requested, stats.bytes_read) == (64, 4096) and np.array_equal(rows[0], m[0])
    stats = IoStats()
    rows = fetch_rows(store, np.arange(64), None, stats)
    assert stats.bytes_read == 4096 and rows.tobytes() == m[:64].tobytes()
    assert page_runs(np.array([0, 64]), 64, 4096) == ([(0, 2)], 2)
    assert page_runs(np.array([0, 128]), 64, 4096) == ([(0, 1), (2, 1)], 2)
    w = kb.synth.uniform(10, 300, 2)  # 2400-byte rows: row 1 spans pages 0 and 1
    w.tofile(tmp_path / "s.raw")
    with RowStore(tmp_path / "s.raw", 10, 300) as s2:
        stats = IoStats()
        assert np.array_equal(fetch_rows(s2, np.array([1]), None, stats)[0], w[1])
        assert stats.bytes_read == 8192


def test_fetch_validates_and_store_errors(tmp_path, store_8):
    store, m = store_8
    with pytest.raises(IndexError):
        fetch_rows(store, np.array([512]))
    with pytest.raises(ValueError, match="ascending"):
        fetch_rows(store, np.array([5, 3]))
    (tmp_path / "w.raw").write_bytes(b"\x00" * 100)
    with pytest.raises(kb.MatrixFormatError, match="expected"):
        RowStore(tmp_path / "w.raw", 4, 4)
    with pytest.raises(ValueError, match="page_size"):
        RowStore(tmp_path / "w.raw", 5, 2, page_size=0)
    h = kb.synth.uniform(100, 4, 9)
    kb.save_matrix(h, tmp_path / "h.knrm")
    with RowStore.open(tmp_path / "h.knrm") as s3:
        assert (s3.n, s3.d) == (100, 4)
        assert fetch_rows(s3, np.arange(100)).tobytes() == h.tobytes()
        out = np.empty((100, 4))
        s3.read_all_into(out, chunk_bytes=1000)
        assert out.tobytes() == h.tobytes()
    m.tofile(tmp_path / "t.raw")
    s4 = RowStore(tmp_path / "t.raw", 512, 8)
    with open(tmp_path / "t.raw", "r+b") as fh:
        fh.truncate(1000)
    with pytest.raises(kb.MatrixFormatError, match="page"):
        fetch_rows(s4, np.arange(512))
    s4.close()


def test_refresh_schedule():
    assert [t for t in range(1, 80) if should_refresh(t, CacheSchedule(5))] == [5, 15, 35, 75]
    assert [t for t in range(1, 16) if should_refresh(t, CacheSchedule(1))] == [1, 3, 7, 15]
    assert all(OC.should_refresh(t, s) == should_refresh(t, CacheSchedule(s)) for s in (1, 2, 5) for t in range(200))
    with pytest.raises(ValueError, match="refresh start"):
        CacheSchedule(0)
    assert rows_per_partition(4 * 64, 2, 64) == 2


def test_kmeans_ondisk_mode_checks(store_8):
    store, _ = store_8
    with pytest.raises(ValueError, match="sem mode"):
        kmeans_ondisk(store, kb.EngineConfig(k=2))
    with pytest.raises(ValueError, match="kmeans_ondisk"):
        kb.kmeans(np.zeros((4, 2)), kb.EngineConfig(k=2, mode="sem"))
    with pytest.raises(ValueError, match="capacity"):
        kmeans_ondisk(store, kb.EngineConfig(k=2, mode="sem"), cache_capacity=-1)


def test_row_cache_rebuild_truncates_by_ascending_id():
    """outofcore.py RowCache semantics (test_sem.py's cache case)."""
    cache = kb.RowCache(n_partitions=2, capacity_bytes=4 * 64, row_bytes=64)
    assert cache.rows_per_partition == 2
    rows = np.random.default_rng(0).normal(size=(6, 8))
    cache.rebuild([[(np.array([5, 9]), rows[0:2]), (np.array([1]), rows[2:3])],
                   [(np.array([20, 30, 40]), rows[3:6])]])
    assert sorted(cache.published) == [1, 5, 20, 30]
    assert cache.cached_bytes() <= cache.capacity_bytes
    assert np.array_equal(cache.published[1], rows[2])
    assert cache.cached_rows() == 4


def test_fetch_rows_through_a_cache(tmp_path):
    m = kb.synth.uniform(256, 8, 1)
    m.tofile(tmp_path / "c.raw")
    cache = kb.RowCache(1, 64 * 64, 64)
    cache.rebuild([[(np.arange(0, 64), m[:64])]])
    with RowStore(tmp_path / "c.raw", 256, 8) as store:
        stats = IoStats()
        rows = fetch_rows(store, np.array([3, 10, 100, 200]), cache, stats)
    assert rows.tobytes() == m[[3, 10, 100, 200]].tobytes()
    assert (stats.cache_hits, stats.cache_misses) == (2, 2)
    assert stats.bytes_read == 2 * 4096 and stats.bytes_requested == 4 * 64
