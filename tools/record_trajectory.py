"""Record a full-size GPU trajectory for the step-wise parity goldens (SURVEY.md 8(c):
"C4/C5: step-wise + sampled").

TEST INFRASTRUCTURE.  Runs BASELINE config c4 (856M x 16, PCG64 rows generated in HBM) or
c5 (10M x 256 f32, the numpy mixture law of synth.mixture) on one B200, one pass at a
time, and saves the centroids every pass used, the per-pass statistics and the
assignments of a few row shards at selected passes:

    python tools/record_trajectory.py c4 gpurun_out/traj_c4.npz

oracle/make_golden_stepwise.py then runs the REFERENCE on those shards with those
centroids in the build container; tests/test_gpu_stepwise.py replays the run and
checks both.
"""
from __future__ import annotations

import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1606_08905_b200 as kb  # noqa: E402

SHARD = 4096
PLAN = {
    "c4": dict(steps=(0, 10, 19), shards=lambda n: [0, n // 2 - SHARD // 2, n - SHARD]),
    "c5": dict(steps=(0, 5, 9), shards=lambda n: [0, n // 2 - SHARD // 2, n - SHARD]),
}


def data(name):
    c = kb.synth.CONFIGS[name]
    if name == "c4":
        return kb.synth.uniform_device(c["n"], 16, 4)
    m = c["data"](c["n"])  # numpy law (float32)
    return torch.from_numpy(m).cuda()


def main(name, out):
    c = kb.synth.CONFIGS[name]
    t0 = time.time()
    x = data(name)
    torch.cuda.synchronize()
    print(f"{name}: data {time.time() - t0:.1f}s", flush=True)
    cfg = kb.EngineConfig(k=c["k"], init=c["init"], seed=int(name[1:]), pruning=c["pruning"],
                          max_iters=c["max_iters"], tolerance=c["tolerance"])
    run = kb.Lloyd(x, cfg)
    plan = PLAN[name]
    offs = plan["shards"](c["n"])
    cents, shard_assign = [], {}
    t = 0
    while True:
        cents.append(run.ctx.centroids()[0])
        run.step()
        if t in plan["steps"]:
            a = run.ctx.assignments()
            shard_assign[t] = np.stack([a[o:o + SHARD] for o in offs])
        t += 1
        if run.ctx.state()["stop"]:
            break
    stats = run.ctx.stats()
    means, prev, counts, drift = run.ctx.centroids()
    run.close()
    np.savez_compressed(
        out, name=np.array(name), centroids=np.stack(cents), steps=np.array(plan["steps"]),
        shard_offsets=np.array(offs), shard_rows=np.array(SHARD),
        shard_assign=np.stack([shard_assign[s] for s in plan["steps"]]).astype(np.int32),
        reassignments=np.array([s.reassignments for s in stats]), skips=np.array([s.skips for s in stats]),
        wcss=np.array([s.wcss for s in stats]), means=means, counts=counts,
        init_rows=np.array(run.init_rows if run.init_rows is not None else []))
    print(f"{name}: {len(stats)} passes recorded in {time.time() - t0:.1f}s -> {out}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
