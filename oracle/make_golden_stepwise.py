"""Step-wise parity goldens for BASELINE configs c4 and c5 at their full sizes.

TEST INFRASTRUCTURE ONLY.  SURVEY.md section 8(c): C4 (110 GB) and C5 (10 GB, 3 h of
reference time) cannot be run whole by the reference in this container, so the check is
step-wise: a GPU run records the centroids C_t every pass used and the assignments of
three 4096-row shards at a few passes (tools/record_trajectory.py, on a B200); here the
REFERENCE package assigns the same shard rows against the same C_t:

    kmeans(shard, EngineConfig(k, init="given", initial_centroids=C_t, max_iters=1,
                               pruning=False))        # engine.py:489-500

and the fixture keeps its assignments, a near-tie mask (oracle best / second-best gap
below EPS), and a sha256 of every C_t (the GPU test replays the run and
must reproduce them bit for bit).  Shard rows are regenerated exactly: c4 by PCG64
jump-ahead (default_rng(4), advance(row * 16)), c5 from the full numpy mixture stream.

    PYTHONPATH=/root/reference/pkg/src:. python oracle/make_golden_stepwise.py \
        gpurun_out/traj_c4.npz gpurun_out/traj_c5.npz
"""
from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from oracle.lloyd import lloyd_step  # noqa: E402
from paper_1606_08905_b200 import synth  # noqa: E402

OUT = os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "full")
EPS = {"c4": 1e-9, "c5": 1e-4}


def c4_rows(off, rows):
    bg = np.random.PCG64(np.random.SeedSequence(4))
    bg.advance(off * 16)
    return np.random.Generator(bg).random((rows, 16))


def main(paths):
    from numakmeans import EngineConfig, kmeans  # the reference itself

    for path in paths:
        tr = np.load(path)
        name = str(tr["name"])
        c = synth.CONFIGS[name]
        offs = [int(o) for o in tr["shard_offsets"]]
        rows = int(tr["shard_rows"])
        if name == "c4":
            shards = [c4_rows(o, rows) for o in offs]
            full = np.random.default_rng(4).random((offs[0] + rows, 16))[offs[0]:]
            assert np.array_equal(full, shards[0])  # jump-ahead == the sequential stream
        else:
            m = c["data"](c["n"])
            shards = [np.ascontiguousarray(m[o:o + rows]) for o in offs]
            del m
        steps = [int(s) for s in tr["steps"]]
        ref, tie = [], []
        for si, t in enumerate(steps):
            cent = tr["centroids"][t]
            ra, ta = [], []
            for sh in shards:
                res = kmeans(sh, EngineConfig(k=c["k"], init="given", initial_centroids=cent, max_iters=1,
                                              pruning=False))
                ra.append(res.assignments.astype(np.int32))
                _, d1, d2 = lloyd_step(sh.astype(np.float64), cent)
                ta.append((d2 - d1) / np.maximum(d2, 1e-300) < EPS[name])
            ref.append(np.stack(ra))
            tie.append(np.stack(ta))
            agree = np.mean(np.stack(ra) == tr["shard_assign"][si])
            print(f"{name} pass {t}: reference vs recorded GPU shard assignments agree on {agree:.6f} "
                  f"({int(np.stack(ta).sum())} near-ties)", flush=True)
        sha = [hashlib.sha256(np.ascontiguousarray(ct).tobytes()).hexdigest() for ct in tr["centroids"]]
        os.makedirs(OUT, exist_ok=True)
        np.savez_compressed(os.path.join(OUT, f"{name}_steps.npz"), steps=np.array(steps),
                            shard_offsets=np.array(offs), shard_rows=np.array(rows),
                            ref_assign=np.stack(ref), near_tie=np.stack(tie), centroid_sha=np.array(sha),
                            reassignments=tr["reassignments"], skips=tr["skips"], wcss=tr["wcss"],
                            counts=tr["counts"], eps=np.array(EPS[name]))


if __name__ == "__main__":
    main(sys.argv[1:])
