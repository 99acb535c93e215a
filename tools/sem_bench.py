"""Semi-external runs at BASELINE sizes: steady-state iteration time with the rows in
host memory and the HBM row cache at several capacities (the reference's policy:
refresh at start, 3 start, 7 start, ...), against the same run with rows in HBM.

    python tools/sem_bench.py [c2|c3 ...]
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1606_08905_b200 as kb  # noqa: E402

START = 2
for name in [a for a in sys.argv[1:] if not a.startswith("-")] or ["c2", "c3"]:
    cfg = kb.synth.CONFIGS[name]
    m = cfg["data"](cfg["n"])
    n, d = m.shape
    ec = dict(k=cfg["k"], init=cfg["init"], seed=int(name[1:]), pruning=cfg["pruning"], max_iters=60)
    caps = (None, 64 << 20, m.nbytes // 4, m.nbytes // 2, m.nbytes)
    if "--full-only" in sys.argv:
        caps = (m.nbytes,)
    runs = [("hbm", None)] + [(f"sem cap {c}", c) for c in caps]
    for label, cap in runs:
        sem = None
        if label != "hbm":
            sem = dict(T=1, task_size=8192, page_size=4096, cache_enabled=cap is not None,
                       cache_capacity=cap or 0, refresh_start=START)
        r = kb.Lloyd(m, kb.EngineConfig(host_rows=sem is not None, **ec), ignore_stop=True, sem=sem)
        r.ctx.enqueue(8)  # past the refreshes at 2 and 6
        torch.cuda.synchronize()
        K = 6
        t0 = time.perf_counter()
        r.ctx.enqueue(K)
        r.sync()
        el = (time.perf_counter() - t0) / K
        extra = ""
        if sem is not None:
            io = r.ctx.sem_io(8 + K)[8:]
            hits, miss = io[:, 2].sum(), io[:, 3].sum()
            extra = (f"  requested {io[:, 0].mean() / 1e6:.1f} MB/iter  hit rate "
                     f"{hits / max(1, hits + miss):.3f}  link {io[:, 3].mean() * d * 8 / 1e6 if cap else io[:, 0].mean() / 1e6:.1f} MB/iter")
        print(f"{name} {label:>22}: {el * 1e3:8.3f} ms/iter  {n / el / 1e9:6.2f} G pt-it/s{extra}", flush=True)
        r.close()
