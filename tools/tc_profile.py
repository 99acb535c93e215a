"""A few pruned passes of a config-4-shaped problem on the tcgen05 MTI kernel (for ncu).

usage: python tools/tc_profile.py [n] [mode]   (mode: tc | block | auto)"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1606_08905_b200 as kb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20_000_000
mode = sys.argv[2] if len(sys.argv) > 2 else "tc"
x = kb.synth.uniform_device(n, 16, 4)
r = kb.Lloyd(x, kb.EngineConfig(k=100, init="forgy", seed=4, pruning=True, max_iters=10, mti_scan=mode),
             ignore_stop=True)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for i in range(6):
    if i == 3:
        ev[0].record()
    r.step()
ev[1].record()
torch.cuda.synchronize()
st = r.ctx.stats()
print(f"{mode}: n={n} {ev[0].elapsed_time(ev[1]) / 3:.3f} ms/iter, info {r.ctx.mti_tc_info()}, "
      f"moved per pass {[round(s.reassignments / n, 4) for s in st]}")
r.close()
