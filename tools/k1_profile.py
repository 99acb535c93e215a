"""One dense pass of a config-4-shaped problem (for ncu)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1606_08905_b200 as kb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20_000_000
d, k = int(sys.argv[3]) if len(sys.argv) > 3 else 16, int(sys.argv[4]) if len(sys.argv) > 4 else 100
x = kb.synth.uniform_device(n, d, 4)
r = kb.Lloyd(x, kb.EngineConfig(k=k, init="forgy", seed=4, pruning=False, max_iters=6), ignore_stop=True)
for _ in range(4):
    r.step()
torch.cuda.synchronize()
r.close()
