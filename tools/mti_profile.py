"""A few pruned iterations of a config-3-shaped problem (for ncu)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1606_08905_b200 as kb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16_000_000
cfg = kb.synth.CONFIGS["c3"]
x = torch.from_numpy(cfg["data"](n)).cuda()
r = kb.Lloyd(x, kb.EngineConfig(k=10, init="forgy", seed=3, pruning=True, max_iters=8), ignore_stop=True)
for _ in range(6):
    r.step()
torch.cuda.synchronize()
r.close()
