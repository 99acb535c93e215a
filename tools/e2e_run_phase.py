"""Config 4's run phase with and without the output prefetch thread (does the page-touching
worker overlap the device iterations?)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1606_08905_b200 as kb  # noqa: E402
from paper_1606_08905_b200 import _native  # noqa: E402
from paper_1606_08905_b200.centroids import device_init  # noqa: E402
from paper_1606_08905_b200.engine import _prefetch_output, _touched_int32  # noqa: E402
from paper_1606_08905_b200.parallel import LocalComm  # noqa: E402

cfg = kb.synth.CONFIGS["c4"]
n, d = cfg["n"], 16
x = kb.synth.uniform_device(n, d, 4)
ec = kb.EngineConfig(k=cfg["k"], init="forgy", seed=4, pruning=True, max_iters=20, tolerance=0)
t0 = time.perf_counter()
a = _touched_int32(n)
print("touch alone %.0f ms" % (1e3 * (time.perf_counter() - t0)))
del a
for mode in ("no prefetch", "prefetch", "no prefetch", "prefetch"):
    ctx = _native.Context(0, n, n, 0, d, ec.k, True, 20, 0.0, None)
    ctx.attach(x.data_ptr())
    device_init(ctx, LocalComm(), None, "forgy", ec.k, 4, None, n, 0, n, d)
    ctx.sync()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pool, fut = _prefetch_output(n) if mode == "prefetch" else (None, None)
    done = ctx.run(16)
    t1 = time.perf_counter()
    buf = fut.result() if fut else None
    t2 = time.perf_counter()
    out = ctx.assignments(out=buf)
    t3 = time.perf_counter()
    print(f"{mode:12s} run {1e3 * (t1 - t0):7.1f} ms  wait-for-buffer {1e3 * (t2 - t1):6.1f} ms  "
          f"assignments D2H {1e3 * (t3 - t2):6.1f} ms  ({done} iterations)")
    if pool:
        pool.shutdown()
    ctx.close()
    del out, buf
