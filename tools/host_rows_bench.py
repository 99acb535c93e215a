"""Rows left in host memory (knb_attach_host_rows): steady-state iteration time and the
link traffic per iteration (rows scored x row bytes; clause-1 skips never cross)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1606_08905_b200 as kb  # noqa: E402

for name in sys.argv[1:] or ["c2", "c3"]:
    cfg = kb.synth.CONFIGS[name]
    m = cfg["data"](cfg["n"])
    ec = dict(k=cfg["k"], init=cfg["init"], seed=int(name[1:]), pruning=cfg["pruning"], max_iters=40)
    r = kb.Lloyd(m, kb.EngineConfig(host_rows=True, **ec), ignore_stop=True)
    r.ctx.enqueue(5)
    torch.cuda.synchronize()
    K = 20
    t0 = time.perf_counter()
    r.ctx.enqueue(K)
    r.sync()
    el = (time.perf_counter() - t0) / K
    st = r.ctx.stats()[5:5 + K]
    rows = np.mean([s.dist_comps / cfg["k"] for s in st])
    gb = rows * m.shape[1] * 8 / 1e9
    print(f"{name}: host rows {el * 1e3:.3f} ms/iter  {cfg['n'] / el / 1e9:.2f} G pt-it/s  "
          f"link {gb:.3f} GB/iter = {gb / el:.1f} GB/s  skipped {np.mean([s.skips for s in st]) / cfg['n']:.2f}",
          flush=True)
    r.close()
