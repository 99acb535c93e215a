"""Wall-time phases of one kmeans() call (where the e2e leg's time goes)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1606_08905_b200 as kb  # noqa: E402
from paper_1606_08905_b200 import _native  # noqa: E402
from paper_1606_08905_b200.centroids import device_init  # noqa: E402
from paper_1606_08905_b200.parallel import LocalComm  # noqa: E402
from paper_1606_08905_b200.engine import _prefetch_output  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = kb.synth.CONFIGS[name]
if name == "c4":  # as bench.py: generated in HBM, then an ordinary pageable copy
    host = kb.synth.uniform_device(cfg["n"], 16, 4).cpu().numpy()
    torch.cuda.empty_cache()
elif "spec" in cfg:  # config 5: the law generated in HBM, copied to pinned host memory
    dev = kb.synth.mixture_device(cfg["spec"](cfg["n"]))
    pinned = torch.empty(tuple(dev.shape), dtype=dev.dtype, pin_memory=True)
    pinned.copy_(dev)
    del dev
    host = pinned.numpy()
else:
    m = cfg["data"](cfg["n"])
    pinned = torch.empty(m.shape, dtype=torch.float64, pin_memory=True)
    pinned.copy_(torch.from_numpy(m))
    host = pinned.numpy()
ec = kb.EngineConfig(k=cfg["k"], init=cfg["init"], seed=int(name[1:]), pruning=cfg["pruning"],
                     max_iters=cfg["max_iters"], tolerance=cfg["tolerance"])
kb.kmeans(host[:100000], ec)
_native.reserve_staging(0)
for rep in range(2):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    n, d = host.shape
    ctx = _native.Context(0, n, n, 0, d, ec.k, ec.pruning, ec.max_iters, ec.tolerance, None)
    t.append(time.perf_counter())
    (ctx.upload_f32 if host.dtype == np.float32 else ctx.upload)(host)
    t.append(time.perf_counter())
    bad = ctx.first_nonfinite_row()
    t.append(time.perf_counter())
    device_init(ctx, LocalComm(), None, ec.init, ec.k, ec.seed, None, n, 0, n, d)
    ctx.sync()
    t.append(time.perf_counter())
    pool, fut = _prefetch_output(n)
    done = ctx.run(ec.batch)
    pin_out = fut.result() if fut else None
    t.append(time.perf_counter())
    st = ctx.stats(); means = ctx.centroids(); a = ctx.assignments(out=pin_out)
    t.append(time.perf_counter())
    ctx.close()
    t.append(time.perf_counter())
    names = ["create", "upload", "finite", "init", f"run({done})", "results", "close"]
    print(" ".join(f"{nm}={1e3 * (t[i + 1] - t[i]):.2f}ms" for i, nm in enumerate(names)), flush=True)
    t0 = time.perf_counter()
    r = kb.kmeans(host, ec)
    print("kmeans() total %.2f ms, %d iterations" % (1e3 * (time.perf_counter() - t0), r.n_iterations))
