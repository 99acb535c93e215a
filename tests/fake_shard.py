"""Test-only stand-in for one GPU shard (``_native.Context``), computed with the oracle.

It lets the multi-rank orchestration of the product (engine._run, device_init,
parallel.*) run under a gloo process group on CPU: row sharding, the per-
iteration exchange, cross-rank kmeans++ sampling, forgy gathers and
random-partition labels.  It is a checker-side double, never importable from
the product package, and follows the device kernels' contract: the local pass
writes the shard's accumulator vector (sums k*d, counts k, sq k, 8 counters)
into the exchange; finish consumes the all-reduced vector.
"""

from __future__ import annotations

import ctypes
from types import SimpleNamespace

import numpy as np

from oracle import lloyd as O

S_REASSIGNED, S_WCSS, S_COMPUTED, S_SKIPS, S_PSTALE, S_PTIGHT = range(6)


class FakeContext:
    def __init__(self, device, n, n_local, row_lo, d, k, pruning, max_iters, tolerance, stream=None):
        self.n, self.n_local, self.row_lo, self.d, self.k = n, n_local, row_lo, d, k
        self.pruning, self.max_iters, self.tol = bool(pruning), max_iters, tolerance
        self.L = k * d + 2 * k + 8
        self.ex = np.zeros(self.L)
        self.stage = np.zeros((k, d))
        self.X = None
        self.d2 = None

    # ---- plumbing
    def exchange_len(self):
        return self.L

    def set_exchange(self, ptr, length):
        self.ex = np.ctypeslib.as_array((ctypes.c_double * length).from_address(ptr))

    def upload(self, rows, lo=0):
        self.X = np.array(rows, dtype=np.float64)

    def first_nonfinite_row(self):
        bad = np.flatnonzero(~np.isfinite(self.X).all(axis=1))
        return int(bad[0]) if bad.size else -1

    def close(self):
        pass

    def set_option(self, option, value):
        self.mti_scan = value

    def sync(self):
        pass

    def state_bytes(self):
        return 0

    # ---- init
    def _install(self, means):
        self.means = np.array(means, dtype=np.float64)
        self.prev = self.means.copy()
        self.drift = np.zeros(self.k)
        self.counts = np.zeros(self.k, dtype=np.int64)
        self.assign = np.zeros(self.n_local, dtype=np.int32)
        self.upper = np.full(self.n_local, np.inf)
        self.tight = np.zeros(self.n_local, dtype=bool)
        self.run_v = np.zeros(self.L)
        self.t, self.stop, self.converged, self.count_error = 0, False, False, False
        self.rows = []

    def set_centroids(self, means):
        self._install(means)

    def init_gather(self, ids):
        ids = list(ids)
        self.ex[: len(ids) * self.d] = 0.0
        for i, g in enumerate(ids):
            if self.row_lo <= g < self.row_lo + self.n_local:
                self.ex[i * self.d:(i + 1) * self.d] = self.X[g - self.row_lo]

    def init_from_exchange(self, first, count):
        self.stage[first:first + count] = self.ex[: count * self.d].reshape(count, self.d)
        if first + count == self.k:
            self._install(self.stage.copy())

    def init_partition_local(self, labels):
        k, d = self.k, self.d
        self.ex[:] = 0.0
        sums = np.zeros((k, d))
        np.add.at(sums, labels, self.X)
        self.ex[: k * d] = sums.ravel()
        self.ex[k * d:k * d + k] = np.bincount(labels, minlength=k)

    def init_partition_finish(self):
        k, d = self.k, self.d
        sums = self.ex[: k * d].reshape(k, d)
        cnt = self.ex[k * d:k * d + k]
        glob = sums.sum(axis=0) / self.n
        means = np.where(cnt[:, None] > 0, sums / np.maximum(cnt, 1)[:, None], glob[None, :])
        self._install(means)

    def kpp_update(self, first):
        c = self.ex[: self.d].copy()
        dd = O.dist_to(self.X, c) ** 2
        self.d2 = dd if first else np.minimum(self.d2, dd)
        return float(self.d2.sum())

    def kpp_psum(self, total):
        p = self.d2 / total
        self.cum = np.cumsum(p)
        return float(self.cum[-1]) if self.cum.size else 0.0

    def kpp_search(self, total, thr):
        return int(min(np.searchsorted(self.cum, thr, side="right"), self.n_local - 1))

    def kpp_release(self):
        self.d2 = None

    # ---- iterations
    def iter_local(self):
        k, d = self.k, self.d
        sums, cnt, sq = np.zeros((k, d)), np.zeros(k), np.zeros(k)
        sc = np.zeros(8)
        full = (not self.pruning) or self.t == 0
        X = self.X
        if full:
            ids, nd = O.nearest(X, self.means) if self.n_local else (np.zeros(0, np.int32), np.zeros(0))
            sc[S_REASSIGNED] = int((ids != self.assign).sum())
            self.assign[:] = ids
            if self.pruning:
                self.upper[:] = nd
                self.tight[:] = True
                sq += np.bincount(ids, weights=O.sqnorms(X), minlength=k)
            else:
                sc[S_WCSS] = float(np.vecdot(nd, nd))
            cnt += np.bincount(ids, minlength=k)
            np.add.at(sums, ids, X)
            sc[S_COMPUTED] = self.n_local * k
        else:
            mv = self.drift[self.assign]  # bound inflation (pruning.py:152-160), applied at the start
            self.upper += mv
            np.logical_and(self.tight, mv == 0.0, out=self.tight)
            skip = self.upper <= self.hmin[self.assign]
            sc[S_SKIPS] = int(skip.sum())
            live = np.flatnonzero(~skip)
            if live.size:
                a_s, u_s, t_s = self.assign[live], self.upper[live], self.tight[live]
                ctr = dict(skips=0, pruned_stale=0, pruned_tight=0, computed=0)
                orig = O.mti_scan(X[live], self.means, self.half, a_s, u_s, t_s, ctr)
                self.assign[live], self.upper[live], self.tight[live] = a_s, u_s, t_s
                moved = np.flatnonzero(a_s != orig)
                sc[S_REASSIGNED] = moved.size
                sc[S_COMPUTED] = ctr["computed"]
                sc[S_PSTALE] = ctr["pruned_stale"]
                sc[S_PTIGHT] = ctr["pruned_tight"]
                if moved.size:
                    rows = X[live][moved]
                    src, dst = orig[moved], a_s[moved]
                    np.add.at(sums, dst, rows)
                    np.subtract.at(sums, src, rows)
                    cnt += np.bincount(dst, minlength=k) - np.bincount(src, minlength=k)
                    w = O.sqnorms(rows)
                    sq += np.bincount(dst, weights=w, minlength=k) - np.bincount(src, weights=w, minlength=k)
        self.ex[: k * d] = sums.ravel()
        self.ex[k * d:k * d + k] = cnt
        self.ex[k * d + k:k * d + 2 * k] = sq
        self.ex[k * d + 2 * k:] = sc

    def iter_finish(self):
        k, d = self.k, self.d
        v = self.ex.copy()
        if self.pruning:
            self.run_v[: k * d + 2 * k] += v[: k * d + 2 * k]
            tot = self.run_v
        else:
            tot = v
        sums = tot[: k * d].reshape(k, d)
        cnt = tot[k * d:k * d + k]
        sq = tot[k * d + k:k * d + 2 * k]
        sc = v[k * d + 2 * k:]
        if int(round(cnt.sum())) != self.n:
            self.count_error = True
        occ = cnt > 0
        new = self.means.copy()
        new[occ] = sums[occ] / cnt[occ, None]
        drift = O.dist_to(new, self.means)
        drift[~occ] = 0.0
        if self.pruning:
            terms = sq[occ] - (sums[occ] ** 2).sum(axis=1) / cnt[occ]
            wcss = float(np.maximum(terms, 0.0).sum())
        else:
            wcss = float(sc[S_WCSS])
        reassigned = int(round(sc[S_REASSIGNED]))
        conv = reassigned <= self.tol
        stop = conv or self.t + 1 >= self.max_iters
        self.rows.append(SimpleNamespace(t=self.t, reassignments=reassigned, wcss=wcss,
                                         dist_comps=int(round(sc[S_COMPUTED])), skips=int(round(sc[S_SKIPS])),
                                         pruned_stale=int(round(sc[S_PSTALE])),
                                         pruned_tight=int(round(sc[S_PTIGHT]))))
        self.prev, self.means, self.drift = self.means, new, drift
        self.counts = np.rint(cnt).astype(np.int64)
        self.converged, self.stop = conv, stop
        self.t += 1
        if self.pruning and not stop:
            self.half, self.hmin = O.half_geometry(self.means)

    def validate(self):
        ids, _, _ = O.lloyd_step(self.X, self.means) if self.n_local else (self.assign, None, None)
        bad_a = np.flatnonzero(ids != self.assign)
        true_d = O.dist_to(self.X, self.means[self.assign])
        bad_b = np.flatnonzero(self.upper + 1e-9 * np.maximum(1.0, true_d) < true_d)
        return (int(bad_a[0]) if bad_a.size else -1, int(bad_b[0]) if bad_b.size else -1)

    def state(self):
        return dict(stop=self.stop, converged=self.converged, t=self.t, count_error=self.count_error)

    def stats(self):
        return list(self.rows)

    def centroids(self):
        return self.means.copy(), self.prev.copy(), self.counts.copy(), self.drift.copy()

    def assignments(self):
        return self.assign.copy()
