"""CPU oracle for the in-memory Lloyd / MTI k-means path of ``numakmeans``.

TEST INFRASTRUCTURE ONLY.  Nothing on the product path imports this module:
it is used by ``tests/`` (as the parity checker), by
``__graft_entry__.smoke()`` (to check one small GPU run) and by ``bench.py``
(the ``cpu_baseline`` leg and ``--impl reference``).  The product path in
``paper_1606_08905_b200`` fails loudly when its CUDA library is missing; it
never falls back to this code.

What it restates (reference = ``/root/reference/pkg/src/numakmeans``):

* the one f64 distance recipe -- exact subtract, ``np.vecdot`` self-contraction,
  ``sqrt`` (``distance.py:28-39``); ascending strict-less nearest-centroid scan
  (``distance.py:94-116``);
* initialisation: given / forgy / random-partition / kmeans++
  (``centroids.py:131-189``);
* the dense task: nearest, reassignment count, MTI seeding, bincount counts,
  stable-sort segment sums (``engine.py:285-319``);
* the pruned task: clause-1 point skip, tighten, clause-2/3 candidate scan,
  signed deltas (``engine.py:321-354``, ``pruning.py:163-204``);
* the barrier action: pairwise merge by task index, running sums under
  pruning, Sigma counts == n, finalize with the empty-cluster rule and drift,
  WCSS, convergence, bound inflation and centroid geometry
  (``engine.py:358-426``, ``centroids.py:88-128``, ``pruning.py:48-61``,
  ``pruning.py:152-160``);
* row partitioning into T ranges and task blocks (``matrix.py:196-213``,
  ``scheduler.py:152-166``).

Pinning: ``tests/test_oracle_pins.py`` checks this module against the golden
fixtures in ``tests/golden/`` that ``oracle/make_golden.py`` produced by running
the reference package itself in the build container (bit-identical
assignments, per-iteration counters, and centroids), and -- when
``/root/reference`` is mounted -- against the live reference.

The per-task work is fanned out over a thread pool exactly like the
reference's worker threads (numpy ufuncs drop the GIL); task results are
merged in task-index order, so results do not depend on ``threads``.
"""

from __future__ import annotations

import os
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

CHUNK_ELEMS = 262144  # engine.py:56 -- rows per vectorised chunk = CHUNK_ELEMS // d


# ---------------------------------------------------------------------------
# distance recipe (distance.py)


def sq_to(rows: np.ndarray, ref: np.ndarray) -> np.ndarray:
    """Squared distances row-by-row: subtract, then vecdot (distance.py:28-33)."""
    diff = np.subtract(rows, ref)
    return np.vecdot(diff, diff)


def dist_to(rows: np.ndarray, ref: np.ndarray) -> np.ndarray:
    """rowwise_distances (distance.py:36-39)."""
    return np.sqrt(sq_to(rows, ref))


def dist_matrix(rows: np.ndarray, means: np.ndarray) -> np.ndarray:
    """block_distances (distance.py:42-63): (m, k) computed centroid by centroid."""
    out = np.empty((rows.shape[0], means.shape[0]))
    for j in range(means.shape[0]):
        out[:, j] = sq_to(rows, means[j])
    return np.sqrt(out)


def nearest(rows: np.ndarray, means: np.ndarray):
    """Ascending scan with strict-less update, lowest id wins ties (distance.py:94-116)."""
    best = dist_to(rows, means[0])
    ids = np.zeros(rows.shape[0], dtype=np.int32)
    for j in range(1, means.shape[0]):
        dj = dist_to(rows, means[j])
        better = dj < best
        ids[better] = j
        best = np.minimum(best, dj)
    return ids, best


def sqnorms(rows: np.ndarray) -> np.ndarray:
    """row_sqnorms (distance.py:66-72): vecdot(rows, rows), no subtract."""
    return np.vecdot(rows, rows)


# ---------------------------------------------------------------------------
# data checks and partitioning (matrix.py)


class OracleInputError(ValueError):
    pass


def as_matrix(m) -> np.ndarray:
    """check_matrix (matrix.py:35-49): C-contiguous f64, n,d >= 1, all finite."""
    m = np.ascontiguousarray(m, dtype=np.float64)
    if m.ndim != 2:
        raise OracleInputError(f"expected a 2-D matrix, got ndim={m.ndim}")
    if m.shape[0] < 1 or m.shape[1] < 1:
        raise OracleInputError(f"matrix must be at least 1x1, got {m.shape[0]}x{m.shape[1]}")
    finite = np.isfinite(m)
    if not finite.all():
        raise OracleInputError(f"non-finite value in row {int(np.flatnonzero(~finite.all(axis=1))[0])}")
    return m


def row_ranges(n: int, parts: int) -> list[tuple[int, int]]:
    """partition_rows (matrix.py:196-213): sizes differ by <= 1, remainder to low ids."""
    base, rem = divmod(n, parts)
    out, lo = [], 0
    for w in range(parts):
        hi = lo + base + (1 if w < rem else 0)
        out.append((lo, hi))
        lo = hi
    return out


def task_blocks(n: int, T: int, task_size: int) -> list[tuple[int, int]]:
    """enqueue_iteration (scheduler.py:152-166): ranges split into task_size blocks, indexed in order."""
    blocks = []
    for lo, hi in row_ranges(n, T):
        for a in range(lo, hi, task_size):
            blocks.append((a, min(a + task_size, hi)))
    return blocks


# ---------------------------------------------------------------------------
# initialisation (centroids.py:131-189)


def init_means(m: np.ndarray, k: int, method: str, seed: int, initial=None) -> np.ndarray:
    n, d = m.shape
    if method == "given":
        c = np.ascontiguousarray(initial, dtype=np.float64)
        if c.shape != (k, d):
            raise OracleInputError(f"initial centroids must be ({k}, {d}), got {c.shape}")
        return c.copy()
    rng = np.random.default_rng(seed)
    if method == "forgy":
        if k > n:
            raise OracleInputError(f"forgy needs k <= n (k={k}, n={n})")
        return m[np.sort(rng.choice(n, size=k, replace=False))].copy()
    if method == "random-partition":
        perm = rng.permutation(n)
        out = np.empty((k, d))
        for j, grp in enumerate(np.array_split(perm, k)):
            out[j] = m.mean(axis=0) if grp.size == 0 else m[np.sort(grp)].mean(axis=0)
        return out
    if method == "kmeanspp":
        if k > n:
            raise OracleInputError(f"kmeanspp needs k <= n (k={k}, n={n})")
        picks = [int(rng.integers(n))]
        d2 = dist_to(m, m[picks[0]]) ** 2        # sqrt then square (centroids.py:179)
        for _ in range(1, k):
            tot = d2.sum()
            picks.append(int(rng.choice(n, p=d2 / tot)) if tot > 0 else int(rng.integers(n)))
            np.minimum(d2, dist_to(m, m[picks[-1]]) ** 2, out=d2)
        return m[picks].copy()
    raise OracleInputError(f"unknown init method {method!r}")


def kmeanspp_picks(m: np.ndarray, k: int, seed: int) -> list[int]:
    """Row ids chosen by kmeans++ in draw order (same stream as init_means)."""
    n = m.shape[0]
    rng = np.random.default_rng(seed)
    picks = [int(rng.integers(n))]
    d2 = dist_to(m, m[picks[0]]) ** 2
    for _ in range(1, k):
        tot = d2.sum()
        picks.append(int(rng.choice(n, p=d2 / tot)) if tot > 0 else int(rng.integers(n)))
        np.minimum(d2, dist_to(m, m[picks[-1]]) ** 2, out=d2)
    return picks


# ---------------------------------------------------------------------------
# MTI geometry and scan (pruning.py)


def half_geometry(means: np.ndarray):
    """centroid_geometry (pruning.py:48-61): exact half distances, row minima off the diagonal."""
    k = means.shape[0]
    half = np.zeros((k, k))
    for a in range(k - 1):
        h = dist_to(means[a + 1:], means[a]) * 0.5
        half[a, a + 1:] = h
        half[a + 1:, a] = h
    if k == 1:
        return half, np.array([np.inf])
    return half, (half + np.diag(np.full(k, np.inf))).min(axis=1)


def mti_scan(rows, means, half, a, u, tight, ctr):
    """scan_block (pruning.py:163-204) on survivors; a/u/tight updated in place, returns orig ids."""
    stale = u.copy()
    loose = np.flatnonzero(~tight)
    if loose.size:
        u[loose] = dist_to(rows[loose], means[a[loose]])
        ctr["computed"] += int(loose.size)
    tight[:] = True
    orig = a.copy()
    for x in range(means.shape[0]):
        cand = (a != x) & (orig != x)
        if not cand.any():
            continue
        gap = half[a, x]
        cut = cand & (u <= gap)
        nc = int(cut.sum())
        if nc:
            ns = int((cut & (stale <= gap)).sum())
            ctr["pruned_stale"] += ns
            ctr["pruned_tight"] += nc - ns
        todo = np.flatnonzero(cand & ~cut)
        if todo.size == 0:
            continue
        dx = dist_to(rows[todo], means[x])
        ctr["computed"] += int(todo.size)
        win = dx < u[todo]
        if win.any():
            sel = todo[win]
            a[sel] = x
            u[sel] = dx[win]
    return orig


# ---------------------------------------------------------------------------
# engine (engine.py)


@dataclass
class OracleIteration:
    t: int
    reassignments: int
    wcss: float
    dist_comps: int
    skips: int = 0
    pruned_stale: int = 0
    pruned_tight: int = 0
    wall_s: float = 0.0


@dataclass
class OracleResult:
    means: np.ndarray
    prev_means: np.ndarray
    counts: np.ndarray
    drift: np.ndarray
    assignments: np.ndarray
    iterations: list[OracleIteration]
    converged: bool
    history: list[np.ndarray] | None = None
    init_means: np.ndarray | None = None
    upper: np.ndarray | None = None
    tight: np.ndarray | None = None
    fetched: list[np.ndarray] | None = None  # collect_fetch: rows each iteration reads

    @property
    def n_iterations(self) -> int:
        return len(self.iterations)


@dataclass
class _Part:
    sums: np.ndarray
    counts: np.ndarray
    sq: np.ndarray
    reassigned: int = 0
    wcss: float = 0.0
    ctr: dict = field(default_factory=lambda: dict(skips=0, pruned_stale=0, pruned_tight=0, computed=0))


def _tree_merge(parts: list[_Part]) -> _Part:
    """merge_accumulators (centroids.py:88-107): pairs (2i, 2i+1), odd tail carried."""
    level = list(parts)
    while len(level) > 1:
        nxt = []
        for i in range(0, len(level) - 1, 2):
            level[i].sums += level[i + 1].sums
            level[i].counts += level[i + 1].counts
            level[i].sq += level[i + 1].sq
            nxt.append(level[i])
        if len(level) % 2:
            nxt.append(level[-1])
        level = nxt
    return level[0]


class _Run:
    def __init__(self, m, k, pruning, chunk):
        self.m, self.k, self.pruning, self.chunk = m, k, pruning, chunk
        n = m.shape[0]
        self.assign = np.zeros(n, dtype=np.int32)               # engine.py:226
        self.upper = np.full(n, np.inf) if pruning else None    # engine.py:227-232
        self.tight = np.zeros(n, dtype=bool) if pruning else None
        self.means = None
        self.half = None
        self.half_min = None

    def full_block(self, lo, hi) -> _Part:
        """engine.py:285-319."""
        k, d = self.k, self.m.shape[1]
        p = _Part(np.zeros((k, d)), np.zeros(k, dtype=np.int64), np.zeros(k))
        for a in range(lo, hi, self.chunk):
            b = min(a + self.chunk, hi)
            rows = self.m[a:b]
            ids, nd = nearest(rows, self.means)
            p.reassigned += int((ids != self.assign[a:b]).sum())
            self.assign[a:b] = ids
            if self.pruning:
                self.upper[a:b] = nd
                self.tight[a:b] = True
                p.sq += np.bincount(ids, weights=sqnorms(rows), minlength=k)
            else:
                p.wcss += float(np.vecdot(nd, nd))
            p.counts += np.bincount(ids, minlength=k)
            order = np.argsort(ids, kind="stable")
            sid = ids[order]
            heads = np.concatenate(([0], np.flatnonzero(np.diff(sid)) + 1))
            p.sums[sid[heads]] += np.add.reduceat(rows[order], heads, axis=0)
        p.ctr["computed"] = (hi - lo) * k
        return p

    def pruned_block(self, lo, hi) -> _Part:
        """engine.py:321-354."""
        k, d = self.k, self.m.shape[1]
        p = _Part(np.zeros((k, d)), np.zeros(k, dtype=np.int64), np.zeros(k))
        a = self.assign[lo:hi]
        u = self.upper[lo:hi]
        tg = self.tight[lo:hi]
        skip = u <= self.half_min[a]
        p.ctr["skips"] = int(skip.sum())
        live = np.flatnonzero(~skip)
        if live.size == 0:
            return p
        rows = self.m[lo + live]
        a_s, u_s, t_s = a[live], u[live], tg[live]
        orig = mti_scan(rows, self.means, self.half, a_s, u_s, t_s, p.ctr)
        a[live], u[live], tg[live] = a_s, u_s, t_s
        moved = np.flatnonzero(a_s != orig)
        p.reassigned = int(moved.size)
        if moved.size:
            mv = rows[moved]
            src, dst = orig[moved], a_s[moved]
            np.add.at(p.sums, dst, mv)
            np.subtract.at(p.sums, src, mv)
            p.counts += np.bincount(dst, minlength=k) - np.bincount(src, minlength=k)
            w = sqnorms(mv)
            p.sq += np.bincount(dst, weights=w, minlength=k) - np.bincount(src, weights=w, minlength=k)
        return p


def lloyd(m, k: int, *, max_iters: int = 100, init: str = "forgy", seed: int = 0,
          pruning: bool = True, tolerance: float = 0, initial=None, T: int = 1,
          task_size: int = 8192, collect: bool = False, threads: int | None = None,
          init_override: np.ndarray | None = None, force_iters: bool = False,
          collect_fetch: bool = False) -> OracleResult:
    """The in-memory engine end to end (engine.py:211-500), sequential-equivalent.

    ``T``/``task_size`` fix the accumulator granularity exactly as the reference
    does (they change centroid ulps, never assignments); ``threads`` only sets
    how many host threads run the blocks.  ``init_override`` skips the RNG init
    and starts from the given means (used by the sampled step-wise oracle);
    ``force_iters`` keeps iterating after convergence (benchmark arm only).
    ``collect_fetch`` records, per iteration, the rows a semi-external run reads:
    every row on a full pass (task_rows), the clause-1 survivors on a pruned pass
    (rows_by_ids, engine.py:321-334) -- the input of oracle/outofcore.py.
    """
    m = as_matrix(m)
    n, d = m.shape
    if k < 1 or max_iters < 1 or task_size < 1 or T < 1 or tolerance < 0:
        raise OracleInputError("invalid configuration")
    means0 = (np.ascontiguousarray(init_override, dtype=np.float64).copy()
              if init_override is not None else init_means(m, k, init, seed, initial))
    run = _Run(m, k, pruning, max(1, CHUNK_ELEMS // d))
    run.means = means0.copy()
    prev = means0.copy()
    counts = np.zeros(k, dtype=np.int64)
    drift = np.zeros(k)
    if pruning:
        r_sums, r_counts, r_sq = np.zeros((k, d)), np.zeros(k, dtype=np.int64), np.zeros(k)
    blocks = task_blocks(n, T, task_size)
    workers = threads if threads is not None else 1
    pool = ThreadPoolExecutor(max_workers=workers) if workers > 1 else None
    its: list[OracleIteration] = []
    hist = [] if collect else None
    fetched = [] if collect_fetch else None
    converged = False
    full = True
    t = 0
    try:
        while True:
            t_start = time.perf_counter()
            if fetched is not None:
                fetched.append(np.ones(n, dtype=bool) if full else
                               ~(run.upper <= run.half_min[run.assign]))
            fn = run.full_block if full else run.pruned_block
            if pool is None:
                parts = [fn(lo, hi) for lo, hi in blocks]
            else:
                parts = list(pool.map(lambda b: fn(*b), blocks))
            reassigned = sum(p.reassigned for p in parts)
            ctr = {key: sum(p.ctr[key] for p in parts) for key in parts[0].ctr} if parts else \
                dict(skips=0, pruned_stale=0, pruned_tight=0, computed=0)
            wcss_dense = sum(p.wcss for p in parts)
            merged = _tree_merge(parts) if parts else _Part(np.zeros((k, d)), np.zeros(k, dtype=np.int64), np.zeros(k))
            if pruning:
                r_sums += merged.sums
                r_counts += merged.counts
                r_sq += merged.sq
                tot_s, tot_c, tot_q = r_sums, r_counts, r_sq
            else:
                tot_s, tot_c, tot_q = merged.sums, merged.counts, merged.sq
            if int(tot_c.sum()) != n:
                raise RuntimeError(f"iteration {t}: accumulator counts sum to {int(tot_c.sum())}, expected {n}")
            # finalize_centroids (centroids.py:110-128)
            occ = tot_c > 0
            new = np.empty((k, d))
            new[occ] = tot_s[occ] / tot_c[occ, None]
            new[~occ] = run.means[~occ]
            drift = dist_to(new, run.means)
            drift[~occ] = 0.0
            if pruning:  # engine.py:385-388
                terms = tot_q[occ] - (tot_s[occ] ** 2).sum(axis=1) / tot_c[occ]
                wcss = float(np.maximum(terms, 0.0).sum())
            else:
                wcss = wcss_dense
            its.append(OracleIteration(t, reassigned, wcss, ctr["computed"], ctr["skips"],
                                       ctr["pruned_stale"], ctr["pruned_tight"], time.perf_counter() - t_start))
            if hist is not None:
                hist.append(run.assign.copy())
            prev = run.means
            run.means = new
            counts = tot_c.copy()
            converged = reassigned <= tolerance
            if (converged and not force_iters) or t + 1 >= max_iters:
                break
            t += 1
            if pruning:  # inflate_bounds (pruning.py:152-160) + geometry
                mv = drift[run.assign]
                run.upper += mv
                np.logical_and(run.tight, mv == 0.0, out=run.tight)
                run.half, run.half_min = half_geometry(run.means)
                full = False
    finally:
        if pool is not None:
            pool.shutdown()
    return OracleResult(means=run.means, prev_means=prev, counts=counts, drift=drift,
                        assignments=run.assign.copy(), iterations=its, converged=converged,
                        history=hist, init_means=means0, fetched=fetched,
                        upper=None if run.upper is None else run.upper.copy(),
                        tight=None if run.tight is None else run.tight.copy())


def lloyd_step(m, means: np.ndarray):
    """One dense assignment against fixed ``means`` (for the sampled step-wise check).

    Returns (ids, nearest distance, second-nearest distance) computed with the
    reference recipe; the second distance lets a caller measure the best /
    second-best gap that the near-tie epsilon rule is stated in.
    """
    m = as_matrix(m)
    dm = dist_matrix(m, means)
    ids = np.argmin(dm, axis=1).astype(np.int32)
    part = np.partition(dm, 1, axis=1) if means.shape[0] > 1 else np.concatenate([dm, dm], axis=1)
    return ids, part[:, 0], part[:, 1]


def default_threads() -> int:
    return max(1, os.cpu_count() or 1)
