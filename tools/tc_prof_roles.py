"""Per-role cycle breakdown of the tcgen05 MTI kernel (needs a -DKNB_TCX_PROF=1 build:
python -c "from paper_1606_08905_b200 import build; build.build(out='scratch/libprof.so', extra=('-DKNB_TCX_PROF=1',))"
then KNB_LIB=scratch/libprof.so python tools/tc_prof_roles.py [n])."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1606_08905_b200 as kb  # noqa: E402
from paper_1606_08905_b200 import _native  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20_000_000
x = kb.synth.uniform_device(n, 16, 4)
r = kb.Lloyd(x, kb.EngineConfig(k=100, init="forgy", seed=4, pruning=True, max_iters=10, mti_scan="tc"),
             ignore_stop=True)
for i in range(3):
    r.step()
torch.cuda.synchronize()
_native.mti_tc_prof()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
r.step()
ev[1].record()
torch.cuda.synchronize()
en, c = _native.mti_tc_prof()
tiles = (n + 127) // 128
sm = 148
names = ["prod wait x_empty", "prod issue", "mma wait A", "mma wait TMEM", "mma issue", "conv wait x_full",
         "conv wait A slot", "conv work", "epi wait TMEM", "epi keys", "epi wait rows", "epi certify/bound/state",
         "acc rows summed (count)", "epi other", "acc wait records", "acc work"]
print(f"profiling build: {en}; one pass {ev[0].elapsed_time(ev[1]):.3f} ms, {tiles} tiles, {tiles / sm:.0f} per CTA")
for nm, v in zip(names, c):
    print(f"  {nm:28s} {v / tiles:9.0f} cycles per tile (per reporting thread)")
r.close()
