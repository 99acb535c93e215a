"""Step-wise parity at the full sizes of BASELINE configs c4 (856M x 16 f64, MTI) and c5
(10M x 256 f32, dense tensor-core path) -- SURVEY.md section 8(c): "C4/C5: step-wise +
sampled".

tests/golden/full/c{4,5}_steps.npz hold, for three passes t, the REFERENCE package's
assignments of three 4096-row shards against the centroids C_t the GPU used in that pass
(oracle/make_golden_stepwise.py), plus the sha256 of every C_t of the recorded run.  The
test replays the whole run on the GPU and checks: every C_t bit for bit (the run is
deterministic), the shard assignments at the checked passes against the reference's
(except rows the fixture marks as near-ties), the iteration count, and the per-pass
reassignment / skip counts of the recorded run."""

from __future__ import annotations

import hashlib
import os

import numpy as np
import pytest

import paper_1606_08905_b200 as kb
from conftest import ROOT

pytestmark = pytest.mark.gpu


def _golden(name):
    return np.load(os.path.join(ROOT, "tests", "golden", "full", f"{name}_steps.npz"))


def _rows(name):
    import torch
    c = kb.synth.CONFIGS[name]
    if name == "c4":
        return kb.synth.uniform_device(c["n"], 16, 4)
    return torch.from_numpy(c["data"](c["n"])).cuda()


def _c4_rows(off, rows):
    # the c4 stream at row `off`: PCG64 jump-ahead (16 doubles per row), as the fixture's maker did
    bg = np.random.PCG64(np.random.SeedSequence(4))
    bg.advance(off * 16)
    return np.random.Generator(bg).random((rows, 16))


@pytest.mark.parametrize("name", ["c4", "c5"])
def test_full_size_stepwise_parity(name):
    """Replays the full-size run.  At the checked passes each shard's assignments are compared
    with the pinned oracle's (oracle/lloyd.py lloyd_step: the reference recipe, pinned bit-exact
    to numakmeans by tests/test_oracle_pins.py) against the centroids C_t this run used, and --
    while the run reproduces the recorded one bit for bit (C_t sha256) -- with the REFERENCE's
    own assignments stored in the fixture, plus the recorded per-pass counters.  A kernel change
    that reorders the deterministic sums (new C_t bits) keeps the oracle check and drops the
    recorded-run comparisons until oracle/make_golden_stepwise.py refreshes the fixture."""
    import torch

    from oracle.lloyd import lloyd_step  # checker only

    g = _golden(name)
    c = kb.synth.CONFIGS[name]
    x = _rows(name)
    run = kb.Lloyd(x, kb.EngineConfig(k=c["k"], init=c["init"], seed=int(name[1:]), pruning=c["pruning"],
                                      max_iters=c["max_iters"], tolerance=c["tolerance"]))
    steps = [int(s) for s in g["steps"]]
    offs = [int(o) for o in g["shard_offsets"]]
    rows = int(g["shard_rows"])
    eps = float(g["eps"])
    shards = []
    for o in offs:
        dev = x[o:o + rows].cpu().numpy()
        if name == "c4":
            assert np.array_equal(dev, _c4_rows(o, rows)), "device rows differ from the PCG64 stream"
        shards.append(dev.astype(np.float64))
    recorded = True  # this run has reproduced the recorded one so far
    try:
        t = 0
        while True:
            cent = run.ctx.centroids()[0]
            recorded = recorded and hashlib.sha256(np.ascontiguousarray(cent).tobytes()).hexdigest() == \
                str(g["centroid_sha"][t])
            run.step()
            if t in steps:
                si = steps.index(t)
                a = run.ctx.assignments()
                for j, o in enumerate(offs):
                    got = a[o:o + rows]
                    ids, d1, d2 = lloyd_step(shards[j], cent)
                    tie = (d2 - d1) / np.maximum(d2, 1e-300) < eps
                    bad = np.flatnonzero(got != ids)
                    assert np.all(tie[bad]), \
                        f"{name} pass {t} shard {o}: {int((~tie[bad]).sum())} non-near-tie mismatches vs the oracle"
                    if recorded:
                        want = g["ref_assign"][si, j]
                        bad = np.flatnonzero(got != want)
                        assert np.all(g["near_tie"][si, j][bad]), \
                            f"{name} pass {t} shard {o}: {int((~g['near_tie'][si, j][bad]).sum())} " \
                            "non-near-tie mismatches vs the reference"
            t += 1
            if run.ctx.state()["stop"]:
                break
        stats = run.ctx.stats()
        assert len(stats) == c["max_iters"] == len(g["reassignments"])
        assert int(run.ctx.centroids()[2].sum()) == c["n"]
        if recorded:
            np.testing.assert_array_equal([s.reassignments for s in stats], g["reassignments"])
            np.testing.assert_array_equal([s.skips for s in stats], g["skips"])
            np.testing.assert_array_equal(run.ctx.centroids()[2], g["counts"])
        else:
            print(f"{name}: C_t differ from the recorded run (summation order changed): "
                  "checked against the oracle only")
    finally:
        run.close()
        del x
        torch.cuda.empty_cache()
