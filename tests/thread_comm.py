"""TEST INFRASTRUCTURE: the product's communicator interface (parallel.TorchComm) for
W ranks that are threads of ONE process sharing one GPU -- so the real kernels of several
row shards (row_lo > 0) run on the single-GPU test box.  Each collective is a barrier
plus a fixed-order reduction on the host thread of rank 0; the exchange buffers are CUDA
tensors the contexts write into (knb_set_exchange), summed in rank order after a device
synchronisation.  No kernel ever waits on another."""

from __future__ import annotations

import threading


class ThreadGroup:
    def __init__(self, world: int):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots = [None] * world


class ThreadComm:
    cuda = True

    def __init__(self, group: ThreadGroup, rank: int):
        self.g, self.rank, self.world = group, rank, group.world

    def _gather(self, x):
        self.g.slots[self.rank] = x
        self.g.barrier.wait()
        out = list(self.g.slots)
        self.g.barrier.wait()
        return out

    def make_exchange(self, length: int, device):
        import torch
        return torch.zeros(length, dtype=torch.float64, device=torch.device("cuda", device or 0))

    def allreduce_exchange(self, buf) -> None:
        import torch
        torch.cuda.synchronize()
        bufs = self._gather(buf)
        if self.rank == 0:
            total = bufs[0].clone()
            for b in bufs[1:]:
                total += b
            for b in bufs:
                b.copy_(total)
            torch.cuda.synchronize()
        self.g.barrier.wait()

    def allreduce_sum(self, x: float) -> float:
        return float(sum(self._gather(float(x))))

    def allreduce_min_int(self, x: int) -> int:
        return int(min(self._gather(int(x))))

    def allreduce_max_int(self, x: int) -> int:
        return int(max(self._gather(int(x))))

    def allgather_float(self, x: float) -> list[float]:
        return [float(v) for v in self._gather(float(x))]

    def allgather_int(self, x: int) -> list[int]:
        return [int(v) for v in self._gather(int(x))]


def run_ranks(world: int, fn):
    """fn(rank, comm) on `world` threads; returns the results in rank order (re-raises)."""
    group = ThreadGroup(world)
    out, err = [None] * world, [None] * world

    def body(r):
        try:
            out[r] = fn(r, ThreadComm(group, r))
        except BaseException as exc:  # noqa: BLE001 - surfaced below
            err[r] = exc
            group.barrier.abort()

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in err:
        if e is not None and not isinstance(e, threading.BrokenBarrierError):
            raise e
    for e in err:
        if e is not None:
            raise e
    return out
