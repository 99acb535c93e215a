"""cProfile of one warm kmeans() call on config 4's host array (where the e2e leg's host time goes)."""
import cProfile
import pstats
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1606_08905_b200 as kb  # noqa: E402
from paper_1606_08905_b200 import _native  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
cfg = kb.synth.CONFIGS[name]
host = kb.synth.uniform_device(cfg["n"], 16, 4).cpu().numpy() if name == "c4" else cfg["data"](cfg["n"])
torch.cuda.empty_cache()
ec = kb.EngineConfig(k=cfg["k"], init=cfg["init"], seed=int(name[1:]), pruning=cfg["pruning"],
                     max_iters=cfg["max_iters"], tolerance=cfg["tolerance"])
kb.kmeans(host[:100000], ec)
_native.reserve_staging(0)
t0 = time.perf_counter()
kb.kmeans(host, ec)
print("first call %.1f ms" % (1e3 * (time.perf_counter() - t0)))
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
r = kb.kmeans(host, ec)
pr.disable()
print("profiled call %.1f ms, %d iterations" % (1e3 * (time.perf_counter() - t0), r.n_iterations))
pstats.Stats(pr).sort_stats("cumulative").print_stats(22)
