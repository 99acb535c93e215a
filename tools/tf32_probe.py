"""How the tcgen05 kind::tf32 path rounds f32 operands (truncate vs nearest), and the
measured score error relative to the certificate's model on config-5-like data."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1606_08905_b200 as kb  # noqa: E402

d, k = 32, 4
vals = [1.0 + 3 * 2.0 ** -12, 1.0 + 2.0 ** -11, 1.0 + 5 * 2.0 ** -12, 1.0 - 3 * 2.0 ** -13]
m = np.zeros((256, d), dtype=np.float32)
for i, v in enumerate(vals):
    m[i, 0] = v
c = np.zeros((k, d))
c[0, 0] = 1.0
c[1, 1] = 1.0
c[2, 0] = 1.0 + 3 * 2.0 ** -12   # B operand rounding
c[3, 2] = 1.0
s = kb.Lloyd(m, kb.EngineConfig(k=k, init="given", initial_centroids=c, pruning=False, max_iters=2))
out = torch.empty((256, 256), dtype=torch.float32, device="cuda")
e = s.ctx.tc_scores(out.data_ptr())
g = out.cpu().numpy()
for i, v in enumerate(vals):
    print(f"x0={v!r}: score vs c0 (x0 - 0.5) = {g[i, 0]!r}  (truncate -> {np.float32(1.0) - 0.5}, exact {v - 0.5})")
print("x0=1 vs c2 (c0=1+3*2^-12):", g[4, 2] if False else None)
m2 = m.copy(); m2[0, 0] = 1.0
s.close()

# error ratio on a config-5-like sample
n, d, k = 20000, 256, 1000
x = kb.synth.mixture(kb.synth.MixtureSpec(n, d, 1000, 5, "normal", 0, 0, 0.3, None, "float32"))
s = kb.Lloyd(x, kb.EngineConfig(k=k, init="forgy", seed=5, pruning=False, max_iters=4))
for step in range(3):
    s.step()
    out = torch.empty((n, 1024), dtype=torch.float32, device="cuda")
    e = s.ctx.tc_scores(out.data_ptr())
    got = out.cpu().numpy()[:, :k].astype(np.float64)
    means, _, _, _ = s.ctx.centroids()
    xd = x.astype(np.float64)
    want = xd @ means.T - 0.5 * np.einsum("ij,ij->i", means, means)[None, :]
    cn = np.sqrt(np.einsum("ij,ij->i", means, means))
    xn = np.sqrt(np.einsum("ij,ij->i", xd, xd))
    err = np.abs(got - want)
    r1 = err / (xn[:, None] * cn.max())
    r2 = err / (np.abs(xd) @ np.abs(means).T)
    print(f"step {step}: max err/(|x| cmax) = {r1.max():.3e} (e = {e:.3e}),  max err/sum|x_i c_i| = {r2.max():.3e}, "
          f"median {np.median(r2):.3e}")
s.close()
