"""§8(f) f2 on CPU: the semi-external I/O oracle pinned against the reference's own
kmeans_ondisk runs (tests/golden/sem/, made by oracle/make_golden_sem.py), and the
host side of the out-of-core API (RowStore, the refresh schedule, kmeans_ondisk's
argument and memory checks)."""

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
from paper_1606_08905_b200 import outofcore
from paper_1606_08905_b200.outofcore import CacheSchedule, RowStore, kmeans_ondisk

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


@pytest.fixture
def store_8(tmp_path):
    m = kb.synth.uniform(512, 8, 5)  # 64-byte rows, payload exactly 8 pages
    path = tmp_path / "m.raw"
    m.tofile(path)
    with RowStore(path, 512, 8) as store:
        yield store, m


def test_store_shape_checks_and_reads(tmp_path, store_8):
    store, m = store_8
    assert (store.n, store.d, store.row_bytes, store.page_size) == (512, 8, 64, 4096)
    assert store.rows[:64].tobytes() == m[:64].tobytes()
    (tmp_path / "w.raw").write_bytes(b"\x00" * 100)
    with pytest.raises(kb.MatrixFormatError, match="expected"):
        RowStore(tmp_path / "w.raw", 4, 4)
    with pytest.raises(ValueError, match="page_size"):
        RowStore(tmp_path / "w.raw", 5, 2, page_size=0)
    with pytest.raises(kb.MatrixFormatError, match="raw"):
        RowStore.open(tmp_path / "w.raw", raw=True)
    h = kb.synth.uniform(100, 4, 9)
    kb.save_matrix(h, tmp_path / "h.knrm")
    with RowStore.open(tmp_path / "h.knrm") as s3:
        assert (s3.n, s3.d) == (100, 4)
        out = np.empty((100, 4))
        s3.read_all_into(out, chunk_rows=7)
        assert out.tobytes() == h.tobytes()


def test_refresh_schedule():
    """CacheSchedule(s) refreshes at s, 3s, 7s, ... -- the oracle's should_refresh, which
    is pinned to the reference's I/O counters."""
    assert [t for t in range(1, 80) if OC.should_refresh(t, CacheSchedule(5).start)] == [5, 15, 35, 75]
    assert [t for t in range(1, 16) if OC.should_refresh(t, CacheSchedule(1).start)] == [1, 3, 7, 15]
    with pytest.raises(ValueError, match="refresh start"):
        CacheSchedule(0)


def test_kmeans_ondisk_mode_checks(store_8):
    store, _ = store_8
    with pytest.raises(ValueError, match="sem mode"):
        kmeans_ondisk(store, kb.EngineConfig(k=2))
    with pytest.raises(ValueError, match="kmeans_ondisk"):
        kb.kmeans(np.zeros((4, 2)), kb.EngineConfig(k=2, mode="sem"))
    with pytest.raises(ValueError, match="capacity"):
        kmeans_ondisk(store, kb.EngineConfig(k=2, mode="sem"), cache_capacity=-1)


def test_kmeans_ondisk_refuses_payloads_beyond_host_memory(store_8, monkeypatch):
    """The payload is staged in host memory (not streamed from disk): a clear
    MemoryError up front when it cannot fit."""
    store, _ = store_8
    monkeypatch.setattr(outofcore, "_available_host_bytes", lambda: 1000)
    with pytest.raises(MemoryError, match="host memory"):
        kmeans_ondisk(store, kb.EngineConfig(k=2, mode="sem"))
