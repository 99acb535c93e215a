"""Seeded synthetic inputs standing in for the paper's datasets.

The paper's Friendster eigenvector and RM/RU matrices are not
available, so BASELINE.json's five configurations are generated here from a
seed with the shapes, sizes and value distributions it states
(SURVEY.md section 8(d)).  Host generation uses numpy's ``default_rng`` so the
bytes are reproducible anywhere the same numpy runs; it is chunked, which
leaves the stream unchanged (``rng.standard_normal((n, d))`` equals the
concatenation of sequential chunk draws).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class MixtureSpec:
    """A mixture of isotropic Gaussians.

    centers: "uniform" in [lo, hi]^d or "normal" (N(0, I)); sigma: a constant
    or a (lo, hi) range drawn per component; weights: None = equal, else the
    Dirichlet concentration.
    """

    n: int
    d: int
    k: int
    seed: int
    centers: str = "uniform"
    lo: float = -10.0
    hi: float = 10.0
    sigma: float | tuple[float, float] = 1.0
    dirichlet: float | None = None
    dtype: str = "float64"


def mixture(spec: MixtureSpec, chunk_rows: int = 1 << 20, out: np.ndarray | None = None) -> np.ndarray:
    rng = np.random.default_rng(spec.seed)
    if spec.centers == "uniform":
        centers = rng.uniform(spec.lo, spec.hi, (spec.k, spec.d))
    elif spec.centers == "normal":
        centers = rng.standard_normal((spec.k, spec.d))
    else:
        raise ValueError(f"unknown center law {spec.centers!r}")
    if isinstance(spec.sigma, tuple):
        sigma = rng.uniform(spec.sigma[0], spec.sigma[1], spec.k)
    else:
        sigma = np.full(spec.k, float(spec.sigma))
    if spec.dirichlet is None:
        w = np.full(spec.k, 1.0 / spec.k)
    else:
        w = rng.dirichlet(np.full(spec.k, float(spec.dirichlet)))
    labels = rng.choice(spec.k, spec.n, p=w)
    x = out if out is not None else np.empty((spec.n, spec.d), dtype=np.dtype(spec.dtype))
    for a in range(0, spec.n, chunk_rows):
        b = min(a + chunk_rows, spec.n)
        lab = labels[a:b]
        x[a:b] = centers[lab] + sigma[lab, None] * rng.standard_normal((b - a, spec.d))
    return x


def uniform(n: int, d: int, seed: int, chunk_rows: int = 1 << 20, dtype="float64") -> np.ndarray:
    """i.i.d. U[0,1)^d = ``default_rng(seed).random((n, d))`` (config 4's law)."""
    rng = np.random.default_rng(seed)
    x = np.empty((n, d), dtype=dtype)
    for a in range(0, n, chunk_rows):
        b = min(a + chunk_rows, n)
        x[a:b] = rng.random((b - a, d))
    return x


def uniform_device(n: int, d: int, seed: int, row_lo: int = 0, rows: int | None = None, device: int = 0):
    """Rows [row_lo, row_lo + rows) of ``default_rng(seed).random((n, d))`` generated
    in HBM by the PCG64 kernel (bit-identical to the host stream) -> CUDA tensor."""
    import torch

    from . import _native

    rows = n - row_lo if rows is None else rows
    st = np.random.default_rng(seed).bit_generator.state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    m64 = (1 << 64) - 1
    out = torch.empty((rows, d), dtype=torch.float64, device=torch.device("cuda", device))
    with torch.cuda.device(device):
        stream = torch.cuda.current_stream().cuda_stream or 1
        rc = _native.lib().knb_fill_uniform_pcg64(
            ctypes.c_void_p(out.data_ptr()), rows * d, row_lo * d, s >> 64, s & m64, inc >> 64, inc & m64,
            ctypes.c_void_p(stream))
    if rc != 0:
        raise RuntimeError(f"knb_fill_uniform_pcg64 failed ({rc})")
    return out


def mixture_device(spec: MixtureSpec, device: int = 0, chunk_rows: int = 1 << 20):
    """The same mixture law generated in HBM with torch's seeded CUDA generator (the
    bytes differ from ``mixture``'s numpy stream; used where only the law matters and
    host generation would dominate, e.g. config 5's 10 GB at full size)."""
    import torch

    dev = torch.device("cuda", device)
    g = torch.Generator(device=dev).manual_seed(spec.seed)
    dt = getattr(torch, spec.dtype)
    if spec.centers == "uniform":
        centers = spec.lo + (spec.hi - spec.lo) * torch.rand((spec.k, spec.d), generator=g, device=dev,
                                                             dtype=torch.float64)
    elif spec.centers == "normal":
        centers = torch.randn((spec.k, spec.d), generator=g, device=dev, dtype=torch.float64)
    else:
        raise ValueError(f"unknown center law {spec.centers!r}")
    if isinstance(spec.sigma, tuple):
        sigma = spec.sigma[0] + (spec.sigma[1] - spec.sigma[0]) * torch.rand(spec.k, generator=g, device=dev,
                                                                            dtype=torch.float64)
    else:
        sigma = torch.full((spec.k,), float(spec.sigma), device=dev, dtype=torch.float64)
    if spec.dirichlet is None:
        w = torch.full((spec.k,), 1.0 / spec.k, device=dev, dtype=torch.float64)
    else:
        gam = torch._standard_gamma(torch.full((spec.k,), float(spec.dirichlet), device=dev, dtype=torch.float64))
        w = gam / gam.sum()
    x = torch.empty((spec.n, spec.d), dtype=dt, device=dev)
    for a in range(0, spec.n, chunk_rows):
        b = min(a + chunk_rows, spec.n)
        lab = torch.multinomial(w, b - a, replacement=True, generator=g)
        noise = torch.randn((b - a, spec.d), generator=g, device=dev, dtype=torch.float64)
        x[a:b] = (centers[lab] + sigma[lab, None] * noise).to(dt)
    return x


# BASELINE.json configs; seed = config index.
CONFIGS = {
    "c1": dict(n=200_000, d=16, k=8, init="forgy", pruning=False, max_iters=20, tolerance=0,
               data=lambda n: mixture(MixtureSpec(n, 16, 8, 1, "uniform", -10, 10, 1.0, None))),
    "c2": dict(n=2_000_000, d=32, k=32, init="kmeanspp", pruning=True, max_iters=100, tolerance=1e-6,
               data=lambda n: mixture(MixtureSpec(n, 32, 32, 2, "uniform", -5, 5, (0.5, 2.0), 1.0))),
    "c3": dict(n=66_000_000, d=8, k=10, init="forgy", pruning=True, max_iters=50, tolerance=0,
               data=lambda n: mixture(MixtureSpec(n, 8, 10, 3, "uniform", -1, 1, 0.1, 0.5))),
    "c4": dict(n=856_000_000, d=16, k=100, init="forgy", pruning=True, max_iters=20, tolerance=0,
               data=lambda n: uniform(n, 16, 4)),
    "c5": dict(n=10_000_000, d=256, k=1000, init="forgy", pruning=False, max_iters=10, tolerance=0,
               data=lambda n: mixture(MixtureSpec(n, 256, 1000, 5, "normal", 0, 0, 0.3, None, "float32")),
               spec=lambda n: MixtureSpec(n, 256, 1000, 5, "normal", 0, 0, 0.3, None, "float32")),
}
# Note: config 4's n rows are a prefix-consistent stream, so any n' < n gives the
# first n' rows of the full matrix; the mixtures are not prefix-consistent in n
# (labels are drawn before the noise), so sub-scale instances are their own datasets.


def config_data(name: str, n: int | None = None) -> np.ndarray:
    cfg = CONFIGS[name]
    return cfg["data"](cfg["n"] if n is None else n)
