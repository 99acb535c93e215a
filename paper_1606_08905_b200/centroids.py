"""Centroid state and initialisation (numakmeans centroids.py).

``CentroidSet`` is the reference's dataclass (centroids.py:15-52).  The four
init methods keep the reference's RNG consumption exactly -- the host draws the
same numbers from ``np.random.default_rng(seed)`` -- while every O(n d) pass
runs on the GPU shards:

* forgy (centroids.py:157-162): host draws ``sort(choice(n, k, replace=False))``,
  owners gather the rows on device;
* random-partition (:164-173): host draws ``permutation(n)``; the device sums the
  rows of each group and divides (empty group -> global mean);
* kmeans++ (:175-189): host draws ``integers(n)`` then one ``random()`` per step
  (``Generator.choice(n, p)`` consumes exactly one); the device
  keeps d2 = min(d2, dist^2) (sqrt then square, as the reference does), sums it,
  and finds the sampled row by a fixed-order scan of d2 / total;
* given (:147-155): shape and finiteness checks, then upload.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .parallel import group_labels, pick_owner

INIT_METHODS = ("forgy", "random-partition", "kmeanspp", "given")


@dataclass
class CentroidSet:
    """Current and previous centroid positions plus per-centroid drift (centroids.py:15-52)."""

    means: np.ndarray       # (k, d)
    prev_means: np.ndarray  # (k, d)
    counts: np.ndarray      # (k,) int64 members after the last finalize (cluster sizes)
    drift: np.ndarray       # (k,) float64

    @property
    def k(self) -> int:
        return self.means.shape[0]

    @property
    def d(self) -> int:
        return self.means.shape[1]

    @classmethod
    def from_means(cls, means: np.ndarray) -> "CentroidSet":
        means = np.ascontiguousarray(means, dtype=np.float64)
        if means.ndim != 2:
            raise ValueError("centroid means must be a (k, d) array")
        if not np.isfinite(means).all():
            raise ValueError("centroid means must be finite")
        k = means.shape[0]
        return cls(means.copy(), means.copy(), np.zeros(k, dtype=np.int64), np.zeros(k))

    def state_bytes(self) -> int:
        return self.means.nbytes + self.prev_means.nbytes + self.counts.nbytes + self.drift.nbytes


def check_init(method: str, k: int, n: int, d: int, initial) -> np.ndarray | None:
    """Argument checks of init_centroids (centroids.py:142-189), same messages."""
    if method not in INIT_METHODS:
        raise ValueError(f"unknown init method {method!r}")
    if k < 1:
        raise ValueError("k must be >= 1")
    if method == "given":
        if initial is None:
            raise ValueError("init method 'given' requires initial centroids")
        initial = np.ascontiguousarray(initial, dtype=np.float64)
        if initial.shape != (k, d):
            raise ValueError(f"initial centroids must be ({k}, {d}), got {initial.shape}")
        if not np.isfinite(initial).all():
            raise ValueError("initial centroids must be finite")
        return initial
    if method == "forgy" and k > n:
        raise ValueError(f"forgy needs k <= n (k={k}, n={n})")
    if method == "kmeanspp" and k > n:
        raise ValueError(f"kmeanspp needs k <= n (k={k}, n={n})")
    return None


def device_init(ctx, comm, exch, method: str, k: int, seed: int, initial, n: int, row_lo: int,
                n_local: int, d: int) -> list[int] | None:
    """Install initial centroids on every shard.  Returns the kmeans++/forgy row ids."""
    initial = check_init(method, k, n, d, initial)
    if method == "given":
        ctx.set_centroids(initial)
        return None
    rng = np.random.default_rng(seed)

    def gather(ids):
        ctx.init_gather(ids)
        comm.allreduce_exchange(exch)

    if method == "forgy":
        ids = np.sort(rng.choice(n, size=k, replace=False))
        gather(ids)
        ctx.init_from_exchange(0, k)
        return [int(i) for i in ids]

    if method == "random-partition":
        labels = group_labels(n, k, rng.permutation(n))
        ctx.init_partition_local(labels[row_lo:row_lo + n_local])
        comm.allreduce_exchange(exch)
        ctx.init_partition_finish()
        return None

    # kmeans++
    if comm.world == 1 and hasattr(ctx, "kpp_run"):
        # one device call: the draws the reference consumes while every D^2 total is > 0
        first = int(rng.integers(n))
        picks, degenerate = ctx.kpp_run(first, rng.random(k - 1))
        if not degenerate:
            ctx.kpp_release()
            return picks
        rng = np.random.default_rng(seed)  # replay the reference's draw order step by step
    picks = [int(rng.integers(n))]
    gather([picks[0]])
    total = comm.allreduce_sum(ctx.kpp_update(first=True))
    for _ in range(1, k):
        if total > 0:
            psums = comm.allgather_float(ctx.kpp_psum(total))
            cdf_end = float(np.sum(psums)) if len(psums) > 1 else psums[0]
            u = rng.random()
            owner, thr = pick_owner(psums, u * cdf_end)
            local = ctx.kpp_search(total, thr) if comm.rank == owner else -1
            bases = comm.allgather_int(row_lo)
            idx = comm.allreduce_max_int(bases[owner] + local if comm.rank == owner else -1)
        else:
            idx = int(rng.integers(n))
        picks.append(idx)
        gather([idx])
        total = comm.allreduce_sum(ctx.kpp_update(first=False))
    gather(picks)
    ctx.init_from_exchange(0, k)
    ctx.kpp_release()
    return picks
