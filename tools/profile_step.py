"""Small driver for ncu: a few iterations of one workload, resident data (no e2e/cpu legs)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1606_08905_b200 as kb

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--iters", type=int, default=4)
ap.add_argument("--dense", action="store_true")
a = ap.parse_args()
cfg = kb.synth.CONFIGS[a.config]
n = a.n or cfg["n"]
m = torch.from_numpy(np.ascontiguousarray(cfg["data"](n), dtype=np.float64)).cuda()
ec = kb.EngineConfig(k=cfg["k"], init=cfg["init"], seed=int(a.config[1:]), pruning=cfg["pruning"] and not a.dense,
                     max_iters=a.iters + 1, tolerance=cfg["tolerance"])
run = kb.Lloyd(m, ec, ignore_stop=True)
for _ in range(a.iters):
    run.step()
run.sync()
st = run.ctx.stats()
print("iters", len(st), "reassign", [s.reassignments for s in st], "comps", [s.dist_comps for s in st])
run.close()
