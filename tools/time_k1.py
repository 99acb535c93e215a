"""Time the steady-state dense local pass (K1) for one config (experiments)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1606_08905_b200 as kb
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = kb.synth.CONFIGS[name]
n = int(sys.argv[2]) if len(sys.argv) > 2 else cfg["n"]
m = torch.from_numpy(np.ascontiguousarray(cfg["data"](n), dtype=np.float64)).cuda()
ec = kb.EngineConfig(k=cfg["k"], init="forgy", seed=1, pruning=False, max_iters=20)
run = kb.Lloyd(m, ec, ignore_stop=True)
run.step(); run.step()
s = torch.cuda.current_stream()
ts = []
for _ in range(8):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s); run.local(); b.record(s); run.finish()
    torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
print(f"{os.environ.get('KNB_LIB','main')}: {name} n={n} K1 local {statistics.median(ts)*1e3:.1f} us")
