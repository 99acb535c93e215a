"""§8(f) f1/f3 on CPU: KNRM files written by the REFERENCE load here, and a report
formatted from the (pinned) oracle's run equals the reference CLI's own report byte for
byte once the timing fields are dropped (tests/golden/reports/, made by
oracle/make_golden_reports.py)."""

from __future__ import annotations

import os
import struct

import numpy as np
import pytest

import paper_1606_08905_b200 as kb
from conftest import ROOT
from oracle import lloyd as O
from oracle import outofcore as OC
from paper_1606_08905_b200.cli import build_parser, config_echo
from paper_1606_08905_b200.engine import IoDelta, IterationStats, KmeansResult
from paper_1606_08905_b200.fileio import HEADER_SIZE, load_matrix, read_header, save_matrix
from paper_1606_08905_b200.report import deterministic_view, format_report, parse_report

GOLD = os.path.join(ROOT, "tests", "golden", "reports")
NAMES = ["kpp_prune", "forgy_dense", "rp_prune_tol", "sem_cache", "sem_nocache_pages", "sem_plain"]


def _args(name):
    with open(os.path.join(GOLD, f"{name}.args")) as fh:
        argv = fh.read().split()
    return build_parser().parse_args(["train", "--data", f"tests/golden/reports/{name}.knrm", *argv])


@pytest.mark.parametrize("name", NAMES)
def test_reference_written_files_load(name):
    path = os.path.join(GOLD, f"{name}.knrm")
    n, d = read_header(path)
    m = load_matrix(path)
    assert m.shape == (n, d) and os.path.getsize(path) == HEADER_SIZE + 8 * n * d
    raw = np.fromfile(path, dtype="<f8", offset=HEADER_SIZE).reshape(n, d)
    assert np.array_equal(np.asarray(m), raw)


@pytest.mark.parametrize("name", NAMES)
def test_report_of_oracle_run_equals_reference_report(name):
    a = _args(name)
    m = np.asarray(load_matrix(os.path.join(ROOT, a.data)))
    o = O.lloyd(m, a.k, init=a.init, seed=a.seed, pruning=a.prune, tolerance=a.tolerance, max_iters=a.max_iters,
                T=a.threads, task_size=a.task_size, collect_fetch=True)
    io = [None] * len(o.iterations)
    if a.mode == "sem":  # the reference's I/O accounting, restated by oracle/outofcore.py
        enabled = True if a.cache is None else a.cache
        cnt = OC.io_counters(o.fetched, [s.skips for s in o.iterations], *m.shape, a.threads, a.task_size,
                             a.page_size, enabled, a.cache_capacity, a.refresh_start)
        io = [IoDelta(*map(int, r)) for r in cnt]
    res = KmeansResult(centroids=None, assignments=o.assignments, converged=o.converged,
                       iterations=[IterationStats(t=s.t, reassignments=s.reassignments, wcss=s.wcss,
                                                  dist_comps=s.dist_comps, skips=s.skips,
                                                  pruned_stale=s.pruned_stale, pruned_tight=s.pruned_tight,
                                                  wall_s=s.wall_s, io=io[i]) for i, s in enumerate(o.iterations)])
    ours = format_report(config_echo(a), res)
    with open(os.path.join(GOLD, f"{name}.report")) as fh:
        ref = fh.read()
    assert deterministic_view(ours) == deterministic_view(ref)
    p = parse_report(ours)
    assert p["totals"]["iters"] == len(o.iterations) and p["converged"] == o.converged
    assert [r["reassign"] for r in p["iterations"]] == [s.reassignments for s in o.iterations]


def test_knrm_round_trip_and_errors(tmp_path):
    m = np.random.default_rng(0).normal(size=(17, 5))
    p = tmp_path / "a.knrm"
    save_matrix(m, p)
    assert np.array_equal(np.asarray(load_matrix(p)), m)
    save_matrix(m, tmp_path / "r.bin", raw=True)
    assert np.array_equal(np.asarray(load_matrix(tmp_path / "r.bin", raw=True, n=17, d=5)), m)
    with pytest.raises(kb.MatrixFormatError, match="raw files carry no shape"):
        load_matrix(tmp_path / "r.bin", raw=True)
    with pytest.raises(kb.MatrixFormatError, match="payload length mismatch"):
        load_matrix(tmp_path / "r.bin", raw=True, n=16, d=5)
    (tmp_path / "short").write_bytes(b"KNRM")
    with pytest.raises(kb.MatrixFormatError, match="too short"):
        load_matrix(tmp_path / "short")
    blob = bytearray(p.read_bytes())
    (tmp_path / "magic").write_bytes(b"XXXX" + bytes(blob[4:]))
    with pytest.raises(kb.MatrixFormatError, match="bad magic"):
        load_matrix(tmp_path / "magic")
    (tmp_path / "ver").write_bytes(blob[:4] + struct.pack("<I", 2) + bytes(blob[8:]))
    with pytest.raises(kb.MatrixFormatError, match="version"):
        load_matrix(tmp_path / "ver")
    bad = m.copy()
    bad[3, 1] = np.nan
    bad.astype("<f8").tofile(tmp_path / "nan.bin")
    with pytest.raises(kb.MatrixFormatError, match="row 3"):
        load_matrix(tmp_path / "nan.bin", raw=True, n=17, d=5)
    with pytest.raises(kb.MatrixIOError):
        load_matrix(tmp_path / "missing.knrm")


def test_cli_info_and_gen(tmp_path, capsys):
    from paper_1606_08905_b200.cli import main
    out = tmp_path / "g.knrm"
    assert main(["gen", str(out), "--family", "gaussian", "--n", "100", "--d", "3", "--k-true", "4"]) == 0
    assert main(["info", str(out)]) == 0
    text = capsys.readouterr().out
    assert "n 100" in text and "d 3" in text and f"file_bytes {HEADER_SIZE + 2400}" in text
    with pytest.raises(SystemExit, match="sem mode only"):
        main(["train", "--data", str(out), "--k", "2", "--cache"])
