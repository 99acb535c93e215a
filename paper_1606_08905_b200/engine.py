"""GPU Lloyd's engine behind the reference API (numakmeans engine.py).

``kmeans(matrix, EngineConfig) -> KmeansResult`` is the drop-in boundary
(engine.py:489-500).  The reference's per-iteration super-phase -- workers
assign and accumulate per task, then one barrier action merges, finalizes and
tests convergence (engine.py:1-23) -- maps onto B200 as:

    knb_iter_local   K1 dense assign+accumulate (full passes) or K6/K7 MTI
                     filter/scan/deltas (pruned passes) over the shard's rows,
                     then the fixed-order merge of CTA partials
    exchange         all-reduce(sum) of the merged vector across GPUs (N > 1)
    knb_iter_finish  running sums, Sigma counts == n, finalize, WCSS, stats row,
                     convergence flag, MTI geometry -- all on device

A single-GPU run without per-iteration host needs (assignment history,
bound validation) queues ``batch`` iterations at a time and reads the device
stop flag between batches; the iteration count and every statistic come from
the device's own stats rows.  There is no CPU fallback.
"""

from __future__ import annotations

import contextlib
import sys
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .centroids import INIT_METHODS, CentroidSet, device_init
from .matrix import MatrixFormatError, check_shape
from .parallel import LocalComm, shard_of

MODES = ("im", "sem")
POLICIES = ("numa", "fifo", "static")


@dataclass
class EngineConfig:
    """Knobs for one clustering run -- the reference's fields and defaults (engine.py:59-96).

    T, N, task_size and scheduler steer the reference's CPU threads; they are
    validated identically and have no effect on GPU results.  Additions:
    ``device`` (CUDA device of a single-GPU run), ``batch`` (iterations queued
    between host checks of the stop flag) and ``mti_scan`` -- how pruned
    iterations re-assign the survivors of the point-skip test: "exact" walks
    candidates with clauses 2/3 like the reference (same dist_comps / pruned_*
    counters), "dense" scores survivors on the FP64 tensor cores (same
    assignments, bounds, skips and centroids; dist_comps = k per survivor,
    pruned_* = 0), "auto" = "dense" where the tensor-core kernel applies.
    ``host_rows``: a host array is not copied to HBM but page-locked and read over
    the host link by every pass (data larger than HBM); pruned passes fetch only
    the survivors of clause 1, and each iteration reports its link traffic in
    ``IterationStats.io`` (rows_elided = skipped rows), like the reference's
    semi-external mode.
    """

    k: int
    max_iters: int = 100
    init: str = "forgy"
    seed: int = 0
    T: int = 1
    N: int = 0
    task_size: int = 8192
    pruning: bool = True
    mode: str = "im"
    tolerance: float = 0
    scheduler: str = "numa"
    initial_centroids: np.ndarray | None = None
    collect_assignments: bool = False
    validate_bounds: bool = False
    device: int | None = None
    batch: int = 16
    mti_scan: str = "auto"
    host_rows: bool = False

    def validate(self) -> None:
        if self.k < 1:
            raise ValueError("k must be >= 1")
        if self.max_iters < 1:
            raise ValueError("max_iters must be >= 1")
        if self.task_size < 1:
            raise ValueError("task_size must be >= 1")
        if self.T < 1:
            raise ValueError("T must be >= 1")
        if self.N < 0:
            raise ValueError("N must be >= 0")
        if self.tolerance < 0:
            raise ValueError("tolerance must be >= 0")
        if self.init not in INIT_METHODS:
            raise ValueError(f"unknown init {self.init!r}")
        if self.mode not in MODES:
            raise ValueError(f"unknown mode {self.mode!r}")
        if self.scheduler not in POLICIES:
            raise ValueError(f"unknown scheduler {self.scheduler!r}")
        if self.batch < 1:
            raise ValueError("batch must be >= 1")
        if self.mti_scan not in _native.MTI_SCAN:
            raise ValueError(f"unknown mti_scan {self.mti_scan!r}")


@dataclass
class IoDelta:
    """I/O counters (engine.py:99-114); in-memory runs report none."""

    bytes_requested: int = 0
    bytes_read: int = 0
    cache_hits: int = 0
    cache_misses: int = 0
    rows_elided: int = 0


@dataclass
class SchedCounters:
    taken_local: int = 0
    stolen_same_node: int = 0
    stolen_remote: int = 0


@dataclass
class IterationStats:
    """What one iteration did (engine.py:124-144).

    ``wcss``: against the centroids current at assignment time for unpruned runs,
    against the updated means (from the running sums) for pruned runs.  ``wall_s``
    of a batched run is the batch's wall time divided evenly over its iterations.
    """

    t: int
    reassignments: int
    wcss: float
    dist_comps: int
    skips: int = 0
    pruned_stale: int = 0
    pruned_tight: int = 0
    wall_s: float = 0.0
    io: IoDelta | None = None
    sched: SchedCounters = field(default_factory=SchedCounters)


@dataclass
class KmeansResult:
    """engine.py:147-159.  For a sharded run ``assignments`` (and the history) hold the
    calling rank's rows [row_lo, row_lo + len)."""

    centroids: CentroidSet
    assignments: np.ndarray
    iterations: list[IterationStats]
    converged: bool
    io_totals: IoDelta | None = None
    peak_state_bytes: int = 0
    assignment_history: list[np.ndarray] | None = None
    row_lo: int = 0
    init_rows: list[int] | None = None
    row_cache: tuple | None = None  # kmeans_ondisk(inspect_cache=True): (ids, rows) of the HBM cache

    @property
    def n_iterations(self) -> int:
        return len(self.iterations)


@contextlib.contextmanager
def _phase(name: str):
    """NVTX range around a host-side phase of a run ("knb:upload", "knb:init", "knb:iterate",
    "knb:results"), for nsys / ncu --nvtx timelines.  Only when the caller's process has
    torch loaded with CUDA up (the numpy-only path never imports torch); a no-op otherwise."""
    torch = sys.modules.get("torch")
    nv = None
    if torch is not None:
        try:
            nv = torch.cuda.nvtx if torch.cuda.is_initialized() else None
        except Exception:
            nv = None
    if nv is None:
        yield
        return
    nv.range_push(name)
    try:
        yield
    finally:
        nv.range_pop()


def torch_stream(device: int) -> int:
    """Handle of torch's current stream on ``device`` for the C ABI; torch's default
    stream reports 0, which is passed as cudaStreamLegacy (0x1) so the library does
    not create a private stream."""
    import torch
    with torch.cuda.device(device):
        h = torch.cuda.current_stream().cuda_stream
    return h or 1


def _rows_of(matrix, cfg: EngineConfig):
    """numpy -> host rows (validated shape); torch CUDA tensor -> device rows (zero copy).

    Rows are f64 like the reference's check_matrix (matrix.py:40), except f32 input on a
    configuration the f32 tensor-core path serves (``_native.f32_supported``): it stays
    f32 -- the reference's upcast is exact, so nothing changes but the bytes moved."""
    try:
        import torch  # noqa: F401
        is_tensor = type(matrix).__module__.startswith("torch")
    except ImportError:  # pragma: no cover
        is_tensor = False

    def keep_f32(dtype_is_f32, d):
        return dtype_is_f32 and not cfg.host_rows and _native.f32_supported(d, cfg.k, cfg.pruning)

    if is_tensor:
        import torch
        t = matrix
        if t.dim() != 2:
            raise MatrixFormatError(f"expected a 2-D matrix, got ndim={t.dim()}")
        if t.shape[0] < 1 or t.shape[1] < 1:
            raise MatrixFormatError(f"matrix must be at least 1x1, got {t.shape[0]}x{t.shape[1]}")
        if not t.is_cuda:
            return _rows_of(t.numpy(), cfg)
        f32 = keep_f32(t.dtype == torch.float32, int(t.shape[1]))
        t = t.to(torch.float32 if f32 else torch.float64).contiguous()
        return None, t
    a = np.asarray(matrix)
    if a.ndim == 2 and keep_f32(a.dtype == np.float32, int(a.shape[1])):
        return check_shape(a, keep_f32=True), None
    return check_shape(a), None


def _apply_options(ctx, cfg: EngineConfig) -> None:
    if cfg.mti_scan != "auto":
        ctx.set_option(_native.KNB_OPT_MTI_SCAN, _native.MTI_SCAN[cfg.mti_scan])
    elif cfg.host_rows and cfg.pruning:
        try:  # compacted survivors: skipped rows never cross the host link
            ctx.set_option(_native.KNB_OPT_MTI_SCAN, _native.MTI_SCAN["dense"])
        except ValueError:
            pass


def _attach_rows(ctx, host, dev, host_rows: bool = False) -> None:
    if dev is not None:
        (ctx.attach_f32 if dev.element_size() == 4 else ctx.attach)(dev.data_ptr())
    elif host.dtype == np.float32:
        ctx.upload_f32(host)
    elif host_rows:
        ctx.attach_host(host)
    else:
        ctx.upload(host)


def _link_io(stats, k: int, d: int) -> list[IoDelta]:
    """Host-row runs: bytes fetched over the link per iteration (rows scored x row bytes)
    and the rows clause 1 kept off the link."""
    out = []
    for s in stats:
        b = (int(s.dist_comps) // max(k, 1)) * d * 8
        out.append(IoDelta(bytes_requested=b, bytes_read=b, rows_elided=int(s.skips)))
    return out


def kmeans(matrix, cfg: EngineConfig) -> KmeansResult:
    """Cluster an in-memory matrix on one B200 (engine.py:489-500).

    ``matrix`` is a host array (copied to HBM) or a CUDA tensor (used in place).
    ``cfg.pruning`` selects the dense engine or the MTI engine; both produce the
    reference's assignments every iteration.
    """
    if cfg.mode != "im":
        raise ValueError("kmeans() runs in-memory; use kmeans_ondisk() for sem mode")
    cfg.validate()
    host, dev = _rows_of(matrix, cfg)
    if dev is not None and cfg.device is not None and int(cfg.device) != dev.device.index:
        raise ValueError(f"EngineConfig.device={cfg.device} but the matrix lives on cuda:{dev.device.index}")
    return _run(host, dev, cfg, LocalComm(), device=cfg.device)


def kmeans_sharded(local_rows, cfg: EngineConfig, comm, n_global: int | None = None,
                   device: int | None = None, context_cls=None) -> KmeansResult:
    """One process per GPU: each rank passes ITS contiguous row shard, in rank order
    (the partition_rows split, matrix.py:196-213, when built with ``shard_of``).

    Rows never leave their GPU; one all-reduce of the accumulator vector per
    iteration crosses NVLink.  Results are identical on every rank except
    ``assignments``, which are the rank's own rows.
    """
    if cfg.mode != "im":
        raise ValueError("kmeans() runs in-memory; use kmeans_ondisk() for sem mode")
    cfg.validate()
    host, dev = _rows_of(local_rows, cfg)
    return _run(host, dev, cfg, comm, device=device, n_global=n_global, context_cls=context_cls)


def _run_sem(host_rows: np.ndarray, cfg: EngineConfig, sem: dict) -> KmeansResult:
    """kmeans_ondisk's engine run (outofcore.py): one GPU, rows in host memory, the
    reference's I/O accounting and HBM row cache configured on the context."""
    host, _ = _rows_of(host_rows, cfg)
    return _run(host, None, cfg, LocalComm(), device=cfg.device, sem=sem)


_PREFAULT_MIN = 1 << 20  # rows: below this the output's page faults cost well under a millisecond


def _touched_int32(n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.int32)
    out.fill(0)  # fault every page in now
    return out


def _prefetch_output(n_local: int):
    """The assignments array of a batched single-GPU run, allocated AND faulted in on a
    worker thread while the device iterates (the host only waits then): the final D2H
    then copies into mapped memory instead of taking a page fault every 4 KB (c3: 264 MB
    of assignments).  Page-locking it instead costs more than it saves for a one-off call
    (cudaHostAlloc pins at ~1.4 GB/s and stalls the host's other CUDA calls).
    Returns (pool, future) or (None, None)."""
    if n_local < _PREFAULT_MIN:
        return None, None
    from concurrent.futures import ThreadPoolExecutor

    pool = ThreadPoolExecutor(max_workers=1)
    return pool, pool.submit(_touched_int32, n_local)


def capture_iteration(ctx, comm, exch):
    """One steady-state iteration -- local pass, the communicator's all-reduce of the
    exchange vector (NCCL), finish -- captured as a CUDA graph on a side stream.  Every
    decision inside (stop gates, MTI kernel choice) is device state, so replaying the
    graph runs as many iterations as there are replays; the stop flag turns the kernels
    of iterations past convergence into no-ops."""
    import torch

    cur = torch.cuda.current_stream()
    side = torch.cuda.Stream()
    side.wait_stream(cur)
    g = torch.cuda.CUDAGraph()
    try:
        with torch.cuda.stream(side):
            with torch.cuda.graph(g, stream=side):
                ctx.set_stream(torch.cuda.current_stream().cuda_stream)
                ctx.iter_local()
                comm.allreduce_exchange(exch)
                ctx.iter_finish()
    finally:
        ctx.set_stream(cur.cuda_stream or None)
    cur.wait_stream(side)
    return g


def _run_graphed(ctx, comm, exch, cfg: EngineConfig) -> int:
    """Multi-GPU iterations with the stop flag on the device: iteration 0 (the full
    pass) eagerly, then ``batch`` replays of the captured iteration between host checks
    (as knb_run does on one GPU).  Returns the iterations run."""
    ctx.iter_local()
    comm.allreduce_exchange(exch)
    ctx.iter_finish()
    if ctx.state()["stop"]:
        return 1
    graph = capture_iteration(ctx, comm, exch)
    while True:
        for _ in range(cfg.batch):
            graph.replay()
        st = ctx.state()
        if st["stop"] or st["count_error"]:
            break
    return len(ctx.stats())


def _run(host, dev, cfg: EngineConfig, comm, device=None, n_global=None, context_cls=None,
         sem: dict | None = None) -> KmeansResult:
    rows = host if host is not None else dev
    n_local, d = int(rows.shape[0]), int(rows.shape[1])
    sizes = comm.allgather_int(n_local)
    if n_global is not None and int(n_global) != sum(sizes):
        raise ValueError(f"shards hold {sum(sizes)} rows, expected n_global={n_global}")
    n = sum(sizes)
    row_lo = sum(sizes[:comm.rank])
    k = cfg.k
    if device is None:
        device = dev.device.index if dev is not None else 0
    stream = None
    if dev is not None or getattr(comm, "cuda", False):
        stream = torch_stream(device)  # NCCL orders its all-reduce after torch's current stream
    cls = context_cls or _native.Context
    ctx = cls(device, n, n_local, row_lo, d, k, cfg.pruning, cfg.max_iters, cfg.tolerance, stream)
    out_pool = None
    try:
        _apply_options(ctx, cfg)
        inspect_cache = False
        if sem is not None:
            sem = dict(sem)
            inspect_cache = bool(sem.pop("inspect_cache", False))
            ctx.sem_configure(**sem)
        exch = comm.make_exchange(ctx.exchange_len(), device)
        if exch is not None:
            ctx.set_exchange(exch.data_ptr(), exch.numel())
        with _phase("knb:upload"):
            _attach_rows(ctx, host, dev, cfg.host_rows)
            bad = ctx.first_nonfinite_row()
        bad_global = comm.allreduce_min_int(row_lo + bad if bad >= 0 else n)
        if bad_global < n:
            raise MatrixFormatError(f"non-finite value in row {bad_global}")
        with _phase("knb:init"):
            init_rows = device_init(ctx, comm, exch, cfg.init, k, cfg.seed, cfg.initial_centroids,
                                    n, row_lo, n_local, d)
        history = [] if cfg.collect_assignments else None
        walls: list[float] = []
        batched = comm.world == 1 and history is None and not cfg.validate_bounds
        graphed = ((comm.world > 1 or getattr(comm, "force_graph", False)) and history is None
                   and not cfg.validate_bounds and getattr(comm, "graph_capture", False))
        if graphed:  # stop flag on the device, one captured iteration replayed (NCCL inside)
            t0 = time.perf_counter()
            with _phase("knb:iterate"):
                done = _run_graphed(ctx, comm, exch, cfg)
            el = time.perf_counter() - t0
            walls = [el / max(done, 1)] * done
        elif batched:
            t0 = time.perf_counter()
            out_pool, out_buf = _prefetch_output(n_local)
            with _phase("knb:iterate"):
                done = ctx.run(cfg.batch)
            el = time.perf_counter() - t0
            walls = [el / max(done, 1)] * done
        else:
            for t in range(cfg.max_iters):
                t0 = time.perf_counter()
                ctx.iter_local()
                comm.allreduce_exchange(exch)
                if cfg.validate_bounds and cfg.pruning:
                    ba, bb = ctx.validate()
                    ba = comm.allreduce_max_int(1 if ba >= 0 else 0)
                    bb = comm.allreduce_max_int(1 if bb >= 0 else 0)
                    if ba:
                        raise AssertionError(f"iteration {t}: stored assignment differs from exhaustive argmin")
                    if bb:
                        raise AssertionError(f"iteration {t}: upper bound below true distance")
                ctx.iter_finish()
                st = ctx.state()
                if st["count_error"]:
                    raise RuntimeError(f"iteration {t}: accumulator counts sum to a value other than {n}")
                if history is not None:
                    history.append(ctx.assignments())
                walls.append(time.perf_counter() - t0)
                if st["stop"]:
                    break
        rows_stats = ctx.stats()
        state = ctx.state()
        if state["count_error"]:
            raise RuntimeError(f"accumulator counts sum to a value other than {n}")
        means, prev, counts, drift = ctx.centroids()
        if sem is not None:
            raw = ctx.sem_io(len(rows_stats))
            io = [IoDelta(bytes_requested=int(r[0]), bytes_read=int(r[1]), cache_hits=int(r[2]),
                          cache_misses=int(r[3]), rows_elided=int(s.skips)) for r, s in zip(raw, rows_stats)]
        elif cfg.host_rows and host is not None:
            io = _link_io(rows_stats, k, d)
        else:
            io = [None] * len(rows_stats)
        its = [IterationStats(t=int(s.t), reassignments=int(s.reassignments), wcss=float(s.wcss),
                              dist_comps=int(s.dist_comps), skips=int(s.skips),
                              pruned_stale=int(s.pruned_stale), pruned_tight=int(s.pruned_tight),
                              wall_s=walls[i] if i < len(walls) else 0.0, io=io[i])
               for i, s in enumerate(rows_stats)]
        io_totals = None
        if io and io[0] is not None:
            io_totals = IoDelta(bytes_requested=sum(x.bytes_requested for x in io),
                                bytes_read=sum(x.bytes_read for x in io),
                                cache_hits=sum(x.cache_hits for x in io),
                                cache_misses=sum(x.cache_misses for x in io),
                                rows_elided=sum(x.rows_elided for x in io))
        row_cache = ctx.sem_cache() if inspect_cache else None
        if out_pool is not None:
            assignments = ctx.assignments(out=out_buf.result())
        else:
            assignments = ctx.assignments()
        peak = ctx.state_bytes()
        return KmeansResult(
            centroids=CentroidSet(means=means, prev_means=prev, counts=counts, drift=drift),
            assignments=assignments,
            iterations=its,
            converged=bool(state["converged"]),
            io_totals=io_totals,
            peak_state_bytes=peak,
            assignment_history=history,
            row_lo=row_lo,
            init_rows=init_rows,
            row_cache=row_cache,
        )
    finally:
        if out_pool is not None:
            out_pool.shutdown(wait=False)
        ctx.close()


class Lloyd:
    """Stepwise handle on one run (benchmarks, step-wise checks): rows stay resident,
    ``step()`` runs exactly one iteration (local pass, exchange, finish).  With a
    ``comm`` each rank passes its own row shard, as in ``kmeans_sharded``."""

    def __init__(self, rows, cfg: EngineConfig, comm=None, ignore_stop: bool = False,
                 device: int | None = None, sem: dict | None = None):
        cfg.validate()
        self.comm = comm or LocalComm()
        host, dev = _rows_of(rows, cfg)
        r = host if host is not None else dev
        self.n_local, self.d = int(r.shape[0]), int(r.shape[1])
        sizes = self.comm.allgather_int(self.n_local)
        self.n = sum(sizes)
        self.row_lo = sum(sizes[:self.comm.rank])
        self.cfg = cfg
        if device is None:
            device = cfg.device if cfg.device is not None else (dev.device.index if dev is not None else 0)
        self.device = device
        stream = None
        if dev is not None or getattr(self.comm, "cuda", False):
            stream = torch_stream(device)
        self.ctx = _native.Context(device, self.n, self.n_local, self.row_lo, self.d, cfg.k, cfg.pruning,
                                   cfg.max_iters, cfg.tolerance, stream)
        _apply_options(self.ctx, cfg)
        if sem is not None:  # semi-external accounting + HBM row cache (knb_sem_configure)
            self.ctx.sem_configure(**sem)
        self._dev = dev
        self.exch = self.comm.make_exchange(self.ctx.exchange_len(), device)
        if self.exch is not None:
            self.ctx.set_exchange(self.exch.data_ptr(), self.exch.numel())
        _attach_rows(self.ctx, host, dev, cfg.host_rows)
        self.init_rows = device_init(self.ctx, self.comm, self.exch, cfg.init, cfg.k, cfg.seed,
                                     cfg.initial_centroids, self.n, self.row_lo, self.n_local, self.d)
        if ignore_stop:
            self.ctx.set_ignore_stop(True)

    def local(self) -> None:
        self.ctx.iter_local()

    def exchange(self) -> None:
        self.comm.allreduce_exchange(self.exch)

    def finish(self) -> None:
        self.ctx.iter_finish()

    def step(self) -> None:
        self.local()
        self.exchange()
        self.finish()

    def sync(self) -> None:
        self.ctx.sync()

    def close(self) -> None:
        self.ctx.close()
