"""Cross-GPU plumbing: one process per GPU, row shards, one exchange per iteration.

The reference's only synchronisation is the per-iteration barrier whose action
merges per-task accumulators (engine.py:253, :358-370; centroids.py:88-107).
Across GPUs that becomes ONE all-reduce(sum) of each shard's merged
accumulator vector (k*d sums, k counts, k squared-norm sums, 8 counters) over
NCCL -- rows never move.  Every rank then finalizes redundantly on identical
inputs, so centroids, drift and the MTI geometry stay bit-identical on all
ranks without a broadcast.

``LocalComm`` is the single-GPU identity.  ``TorchComm`` wraps an initialised
``torch.distributed`` process group (NCCL over NVLink on the GPU box, gloo in
the CPU tests).
"""

from __future__ import annotations

import numpy as np


class LocalComm:
    rank = 0
    world = 1

    def make_exchange(self, length: int, device: int | None):
        return None  # the context's own device buffer is used

    def allreduce_exchange(self, buf) -> None:
        pass

    def allreduce_sum(self, x: float) -> float:
        return float(x)

    def allreduce_min_int(self, x: int) -> int:
        return int(x)

    def allreduce_max_int(self, x: int) -> int:
        return int(x)

    def allgather_float(self, x: float) -> list[float]:
        return [float(x)]

    def allgather_int(self, x: int) -> list[int]:
        return [int(x)]


class TorchComm:
    """torch.distributed process group (NCCL for CUDA tensors, gloo for CPU tests)."""

    def __init__(self, group=None, device: str | None = None):
        import torch
        import torch.distributed as dist

        self.torch, self.dist, self.group = torch, dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        backend = dist.get_backend(group)
        self.cuda = backend == "nccl"
        # NCCL collectives can be captured into a CUDA graph with the local pass and the
        # finish (engine.capture_iteration); gloo's cannot
        self.graph_capture = self.cuda
        self.scalar_device = device or ("cuda" if self.cuda else "cpu")

    def make_exchange(self, length: int, device: int | None):
        t = self.torch
        dev = t.device("cuda", device) if self.cuda else t.device("cpu")
        return t.zeros(length, dtype=t.float64, device=dev)

    def allreduce_exchange(self, buf) -> None:
        self.dist.all_reduce(buf, group=self.group)

    def _scalar(self, x, dtype):
        return self.torch.tensor([x], dtype=dtype, device=self.scalar_device)

    def allreduce_sum(self, x: float) -> float:
        v = self._scalar(float(x), self.torch.float64)
        self.dist.all_reduce(v, group=self.group)
        return float(v.item())

    def allreduce_min_int(self, x: int) -> int:
        v = self._scalar(int(x), self.torch.int64)
        self.dist.all_reduce(v, op=self.dist.ReduceOp.MIN, group=self.group)
        return int(v.item())

    def allreduce_max_int(self, x: int) -> int:
        v = self._scalar(int(x), self.torch.int64)
        self.dist.all_reduce(v, op=self.dist.ReduceOp.MAX, group=self.group)
        return int(v.item())

    def allgather_float(self, x: float) -> list[float]:
        v = self._scalar(float(x), self.torch.float64)
        out = [self.torch.empty_like(v) for _ in range(self.world)]
        self.dist.all_gather(out, v, group=self.group)
        return [float(o.item()) for o in out]

    def allgather_int(self, x: int) -> list[int]:
        v = self._scalar(int(x), self.torch.int64)
        out = [self.torch.empty_like(v) for _ in range(self.world)]
        self.dist.all_gather(out, v, group=self.group)
        return [int(o.item()) for o in out]


def shard_of(n: int, rank: int, world: int) -> tuple[int, int]:
    """[lo, hi) of ``rank`` under the partition_rows rule (matrix.py:196-213)."""
    base, rem = divmod(n, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def pick_owner(psums: list[float], threshold: float) -> tuple[int, float]:
    """Rank whose slice of the kmeans++ CDF contains ``threshold``, and the threshold
    relative to that slice's start (the last rank with mass absorbs rounding)."""
    run = 0.0
    last = max((r for r, p in enumerate(psums) if p > 0), default=len(psums) - 1)
    for r, p in enumerate(psums):
        if p > 0 and (run + p > threshold or r == last):
            return r, threshold - run
        run += p
    return last, threshold - (run - psums[last])


def group_labels(n: int, k: int, perm: np.ndarray) -> np.ndarray:
    """Labels of np.array_split(perm, k) groups (centroids.py:164-173), as one int32 per row."""
    base, rem = divmod(n, k)
    sizes = np.full(k, base, dtype=np.int64)
    sizes[:rem] += 1
    labels = np.empty(n, dtype=np.int32)
    labels[perm] = np.repeat(np.arange(k, dtype=np.int32), sizes)
    return labels
