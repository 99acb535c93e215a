"""Golden-fixture case table shared by oracle/make_golden.py and tests/.

TEST INFRASTRUCTURE ONLY.  Each case names a seeded input (regenerated at test
time -- numpy's Generator streams are stable for a given numpy) and the
``EngineConfig`` fields the reference ran with.  ``make_golden.py`` ran the
reference package on every case in the build container and stored its
outputs under ``tests/golden/<name>.npz``.
"""

from __future__ import annotations

import numpy as np

from paper_1606_08905_b200.synth import MixtureSpec, mixture, uniform


def _hand():
    return np.array([[0.0], [1.0], [10.0], [11.0]])


def _normal(n, d, seed=1234):
    return np.random.default_rng(seed).normal(size=(n, d))


def _tie():
    # every point equidistant from two identical-norm centroids: lowest id must win
    return np.array([[0.0, 0.0], [0.0, 1.0], [0.0, -1.0], [0.0, 2.0], [0.0, 0.5]])


def _tie_pruned(copies: int = 1, d: int = 2):
    """Exact ties between a survivor's CURRENT centroid and a lower id in a pruned pass.

    Per copy: clusters {(-2,0), (-1,0), (-1,2)} and {(1,0), (3,0), (0,2)} (given centroids
    (-1.5, 0.5) and (1, 1.5)); after the first update the means are (-4/3, 2/3) and
    (4/3, 2/3), so (0, 2) -- assigned to the higher id -- is exactly equidistant from both
    and off their segment: it survives clause 1 and clause 2 (u > half_dist), and
    scan_block keeps it (pruning.py:199: switch only on dx < u), while an exhaustive
    lowest-id argmin would move it.  Copies sit 1000 apart on their own axis (dims >= 2)."""
    base = np.array([[-2.0, 0.0], [-1.0, 0.0], [-1.0, 2.0], [1.0, 0.0], [3.0, 0.0], [0.0, 2.0]])
    init = np.array([[-1.5, 0.5], [1.0, 1.5]])
    rows, cents = [], []
    for i in range(copies):
        off = np.zeros(d)
        if copies > 1:
            off[2 + i % (d - 2)] = 1000.0 * (i + 1)
        r = np.zeros((6, d))
        r[:, :2] = base
        c = np.zeros((2, d))
        c[:, :2] = init
        rows.append(r + off)
        cents.append(c + off)
    return np.concatenate(rows), np.concatenate(cents)


CASES = {
    # reference tests' own hand example (test_engine.py:10-22)
    "hand": dict(data=_hand, cfg=dict(k=2, init="given", initial=[[0.0], [10.0]], pruning=False, max_iters=20)),
    "hand_pruned": dict(data=_hand, cfg=dict(k=2, init="given", initial=[[0.0], [10.0]], pruning=True, max_iters=20)),
    "tie": dict(data=_tie, cfg=dict(k=2, init="given", initial=[[-1.0, 0.0], [1.0, 0.0]], pruning=False, max_iters=5)),
    "k1_dense": dict(data=lambda: _normal(100, 3), cfg=dict(k=1, pruning=False, seed=0)),
    "k1_pruned": dict(data=lambda: _normal(100, 3), cfg=dict(k=1, pruning=True, seed=0)),
    "tiny_n3": dict(data=lambda: _normal(3, 2, 77), cfg=dict(k=2, seed=1, pruning=True, max_iters=10)),
    "mix_dense": dict(data=lambda: mixture(MixtureSpec(3000, 4, 6, 21, "uniform", -8, 8, 1.0)),
                      cfg=dict(k=6, seed=4, pruning=False, max_iters=40)),
    "mix_pruned": dict(data=lambda: mixture(MixtureSpec(3000, 4, 6, 21, "uniform", -8, 8, 1.0)),
                       cfg=dict(k=6, seed=4, pruning=True, max_iters=40)),
    "unif_dense": dict(data=lambda: uniform(2000, 3, 21), cfg=dict(k=5, seed=4, pruning=False, max_iters=40)),
    "unif_pruned": dict(data=lambda: uniform(2000, 3, 21), cfg=dict(k=5, seed=4, pruning=True, max_iters=40)),
    "kpp_pruned": dict(data=lambda: mixture(MixtureSpec(5000, 5, 8, 9, "uniform", -6, 6, (0.5, 2.0), 1.0)),
                       cfg=dict(k=8, init="kmeanspp", seed=9, pruning=True, max_iters=30)),
    "rp_dense": dict(data=lambda: mixture(MixtureSpec(3001, 3, 7, 12, "uniform", -5, 5, 1.0)),
                     cfg=dict(k=7, init="random-partition", seed=12, pruning=False, max_iters=30)),
    "rp_empty": dict(data=lambda: _normal(5, 2, 3), cfg=dict(k=8, init="random-partition", seed=3, pruning=False, max_iters=5)),
    "d1_pruned": dict(data=lambda: mixture(MixtureSpec(4000, 1, 5, 31, "uniform", -20, 20, 1.0)),
                      cfg=dict(k=5, seed=31, pruning=True, max_iters=30)),
    "d7_dense": dict(data=lambda: mixture(MixtureSpec(3000, 7, 9, 32, "uniform", -4, 4, 1.0)),
                     cfg=dict(k=9, seed=32, pruning=False, max_iters=30)),
    "d17_pruned": dict(data=lambda: mixture(MixtureSpec(3000, 17, 12, 33, "uniform", -4, 4, 1.0, 1.0)),
                       cfg=dict(k=12, seed=33, pruning=True, max_iters=30)),
    "d33_pruned": dict(data=lambda: mixture(MixtureSpec(2500, 33, 20, 34, "uniform", -3, 3, 1.0)),
                       cfg=dict(k=20, seed=34, pruning=True, max_iters=25)),
    "d65_dense": dict(data=lambda: mixture(MixtureSpec(2000, 65, 16, 35, "uniform", -2, 2, 1.0)),
                      cfg=dict(k=16, seed=35, pruning=False, max_iters=20)),
    "d100_kpp": dict(data=lambda: mixture(MixtureSpec(2000, 100, 10, 36, "normal", 0, 0, 0.3)),
                     cfg=dict(k=10, init="kmeanspp", seed=36, pruning=True, max_iters=20)),
    "k50_pruned": dict(data=lambda: mixture(MixtureSpec(20000, 8, 50, 37, "uniform", -3, 3, 0.5, 1.0)),
                       cfg=dict(k=50, seed=37, pruning=True, max_iters=25)),
    # exact ties with the current centroid in pruned passes: the reference keeps it
    "tie_pruned": dict(data=lambda: _tie_pruned()[0],
                       cfg=dict(k=2, init="given", initial=_tie_pruned()[1], pruning=True, max_iters=10)),
    "tie_pruned_d16": dict(data=lambda: _tie_pruned(12, 16)[0],
                           cfg=dict(k=24, init="given", initial=_tie_pruned(12, 16)[1], pruning=True, max_iters=10)),
    "tie_pruned_d5": dict(data=lambda: _tie_pruned(5, 5)[0],
                          cfg=dict(k=10, init="given", initial=_tie_pruned(5, 5)[1], pruning=True, max_iters=10)),
    # d == DP in {16, 32} with k > 16: the twelve-warp MTI and dense kernels
    "d16_k24_pruned": dict(data=lambda: mixture(MixtureSpec(6000, 16, 24, 38, "uniform", -4, 4, 1.0)),
                           cfg=dict(k=24, seed=38, pruning=True, max_iters=30)),
    "d32_k24_dense": dict(data=lambda: mixture(MixtureSpec(4000, 32, 24, 39, "uniform", -3, 3, 1.0)),
                          cfg=dict(k=24, seed=39, pruning=False, max_iters=25)),
    # BASELINE configs: config 1 in full, the others at reduced n with the same laws
    "c1_full": dict(data=lambda: mixture(MixtureSpec(200_000, 16, 8, 1, "uniform", -10, 10, 1.0)),
                    cfg=dict(k=8, init="forgy", seed=1, pruning=False, max_iters=20, tolerance=0)),
    "c2_mini": dict(data=lambda: mixture(MixtureSpec(20_000, 32, 32, 2, "uniform", -5, 5, (0.5, 2.0), 1.0)),
                    cfg=dict(k=32, init="kmeanspp", seed=2, pruning=True, max_iters=100, tolerance=1e-6)),
    "c3_mini": dict(data=lambda: mixture(MixtureSpec(60_000, 8, 10, 3, "uniform", -1, 1, 0.1, 0.5)),
                    cfg=dict(k=10, init="forgy", seed=3, pruning=True, max_iters=50, tolerance=0)),
    "c4_mini": dict(data=lambda: uniform(20_000, 16, 4),
                    cfg=dict(k=100, init="forgy", seed=4, pruning=True, max_iters=20, tolerance=0)),
    "c5_mini": dict(data=lambda: mixture(MixtureSpec(4000, 256, 1000, 5, "normal", 0, 0, 0.3, None, "float32")),
                    cfg=dict(k=1000, init="forgy", seed=5, pruning=False, max_iters=3, tolerance=0)),
}

# cases cheap enough to rerun through the oracle inside the default CPU suite
FAST = [name for name in CASES if name not in ("c1_full", "c2_mini", "c5_mini", "k50_pruned", "c3_mini")]


def case_data(name: str) -> np.ndarray:
    return CASES[name]["data"]()


def case_cfg(name: str) -> dict:
    cfg = dict(CASES[name]["cfg"])
    if "initial" in cfg:
        cfg["initial"] = np.asarray(cfg["initial"], dtype=np.float64)
    return cfg


# Semi-external runs (kmeans_ondisk, outofcore.py:440-455): data law, EngineConfig
# fields (mode="sem"), and the kmeans_ondisk keywords.  page_size is the RowStore's.
SEM_CASES = {
    "sem_nocache": dict(data=lambda: mixture(MixtureSpec(1600, 8, 4, 19, "uniform", -50, 50, 1.0)),
                        cfg=dict(k=4, seed=3, T=2, max_iters=40),
                        io=dict(cache_enabled=False)),
    "sem_zero_cap": dict(data=lambda: uniform(1500, 6, 3),
                         cfg=dict(k=4, seed=2, T=2, max_iters=40),
                         io=dict(cache_capacity=0, start=1)),
    "sem_quarter": dict(data=lambda: mixture(MixtureSpec(20000, 8, 8, 61, "uniform", -4, 4, 1.0)),
                        cfg=dict(k=8, seed=13, T=2, max_iters=40),
                        io=dict(cache_capacity=20000 * 64 // 4, start=5)),
    "sem_full_s2": dict(data=lambda: uniform(6000, 8, 3),
                        cfg=dict(k=6, seed=2, T=2, max_iters=40),
                        io=dict(cache_capacity=6000 * 64, start=2)),
    "sem_plain_cache": dict(data=lambda: mixture(MixtureSpec(4000, 8, 6, 7, "uniform", -3, 3, 1.0)),
                            cfg=dict(k=6, seed=2, T=3, max_iters=11, pruning=False),
                            io=dict(cache_capacity=4000 * 64 // 2, start=2)),
    "sem_tasks_pages": dict(data=lambda: mixture(MixtureSpec(5000, 8, 7, 23, "uniform", -2, 2, 1.0)),
                            cfg=dict(k=7, seed=4, T=3, task_size=100, max_iters=40),
                            io=dict(cache_capacity=5000 * 64 // 4, start=1, page_size=1000)),
    "sem_wide_rows": dict(data=lambda: uniform(1200, 300, 8),
                          cfg=dict(k=5, seed=1, T=2, max_iters=30),
                          io=dict(cache_capacity=1200 * 2400 // 3, start=2)),
    "sem_kpp_d3": dict(data=lambda: mixture(MixtureSpec(7000, 3, 9, 5, "uniform", -8, 8, 1.0)),
                       cfg=dict(k=9, seed=5, T=4, task_size=333, init="kmeanspp", max_iters=40),
                       io=dict(cache_capacity=7000 * 24 // 10, start=1, page_size=512)),
    "sem_d1": dict(data=lambda: mixture(MixtureSpec(5000, 1, 5, 31, "uniform", -20, 20, 1.0)),
                   cfg=dict(k=5, seed=31, T=1, max_iters=30),
                   io=dict(cache_capacity=5000 * 8 // 4, start=3)),
}


def sem_case(name: str):
    """(matrix, EngineConfig kwargs, kmeans_ondisk kwargs, page_size, refresh start)."""
    c = SEM_CASES[name]
    io = dict(c["io"])
    page = io.pop("page_size", 4096)
    start = io.pop("start", 5)
    return c["data"](), dict(c["cfg"]), io, page, start
