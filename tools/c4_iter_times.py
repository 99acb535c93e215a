"""Per-iteration device time and moved fraction of config 4's first 20 iterations."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1606_08905_b200 as kb  # noqa: E402

cfg = kb.synth.CONFIGS["c4"]
n = int(sys.argv[1]) if len(sys.argv) > 1 else cfg["n"]
x = kb.synth.uniform_device(n, 16, 4)
ec = kb.EngineConfig(k=cfg["k"], init="forgy", seed=4, pruning=True, max_iters=20, tolerance=0)
run = kb.Lloyd(x, ec, ignore_stop=True)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(21)]
s = torch.cuda.current_stream()
ev[0].record(s)
for i in range(20):
    run.step()
    ev[i + 1].record(s)
torch.cuda.synchronize()
st = run.ctx.stats()
for i in range(20):
    print(f"iter {i:2d}: {ev[i].elapsed_time(ev[i + 1]):7.2f} ms  moved {st[i].reassignments / n:6.3f}  skips {st[i].skips}")
run.close()
