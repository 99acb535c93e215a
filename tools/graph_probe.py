"""Timing of graph-replayed iterations (knb_enqueue) vs per-call launches."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1606_08905_b200 as kb  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
cfg = kb.synth.CONFIGS[name]
if name == "c5":
    x = kb.synth.mixture_device(cfg["spec"](cfg["n"]))
else:
    x = torch.from_numpy(cfg["data"](cfg["n"])).cuda()
K = 20
e = kb.EngineConfig(k=cfg["k"], init=cfg["init"], seed=int(name[1:]), pruning=cfg["pruning"], max_iters=200)
r = kb.Lloyd(x, e, ignore_stop=True)
r.step()
r.step()
torch.cuda.synchronize()
s = torch.cuda.current_stream()
for mode in ("calls", "graph", "calls", "graph"):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    a.record(s)
    if mode == "graph":
        r.ctx.enqueue(K)
    else:
        for _ in range(K):
            r.step()
    b.record(s)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(mode, "device ms/step %.4f" % (a.elapsed_time(b) / K), "host enqueue ms/step %.4f" % ((t1 - t0) * 1e3 / K), flush=True)
