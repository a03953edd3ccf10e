"""Ranks emulated by host threads on one GPU (test infrastructure only).

Each thread is one "rank" with its own CUDA stream, contexts, coefficient cache
and reducer.  Collectives synchronise the caller's stream, meet at a host
barrier and combine tensors in rank order; no kernel ever waits on another
kernel, so this is safe on a single device (unlike spinning multi-rank kernels).
"""

import threading

import torch


class _Shared:
    def __init__(self, size):
        self.size = size
        self.barrier = threading.Barrier(size)
        self.slots = [None] * size


class ThreadComm:
    def __init__(self, shared, rank):
        self.sh = shared
        self.rank = rank
        self.size = shared.size
        self.group = None

    def neighbours(self, periodic):
        below = self.rank - 1 if self.rank > 0 else (self.size - 1 if periodic else None)
        above = self.rank + 1 if self.rank < self.size - 1 else (0 if periodic else None)
        return below, above

    def _gather(self, t):
        torch.cuda.current_stream().synchronize()
        self.sh.slots[self.rank] = t.detach().clone()
        self.sh.barrier.wait()
        parts = list(self.sh.slots)
        self.sh.barrier.wait()
        return parts

    def allreduce_sum(self, t):
        parts = self._gather(t)
        tot = parts[0].clone()
        for p in parts[1:]:
            tot += p
        t.copy_(tot)
        return t

    def allreduce_max(self, t):
        parts = self._gather(t)
        tot = parts[0].clone()
        for p in parts[1:]:
            tot = torch.maximum(tot, p)
        t.copy_(tot)
        return t

    def gather_host(self, obj):
        self.sh.barrier.wait()
        self.sh.slots[self.rank] = obj
        self.sh.barrier.wait()
        objs = list(self.sh.slots)
        self.sh.barrier.wait()
        return objs

    def stream_to_root(self, planes, consume, root=0):
        for f in range(len(planes)):
            torch.cuda.current_stream().synchronize()
            self.sh.barrier.wait()
            self.sh.slots[self.rank] = planes[f].detach().cpu().numpy()
            self.sh.barrier.wait()
            if self.rank == root:
                for r in range(self.size):
                    consume(f, r, self.sh.slots[r])
            self.sh.barrier.wait()

    def exchange_rows(self, send_lo, send_hi, recv_lo, recv_hi, periodic):
        torch.cuda.current_stream().synchronize()
        self.sh.slots[self.rank] = (send_lo.clone(), send_hi.clone())
        self.sh.barrier.wait()
        below, above = self.neighbours(periodic)
        if below is not None:
            recv_lo.copy_(self.sh.slots[below][1])
        if above is not None:
            recv_hi.copy_(self.sh.slots[above][0])
        torch.cuda.current_stream().synchronize()
        self.sh.barrier.wait()


def run_ranks(size, fn):
    """Run fn(comm) on `size` thread-ranks; returns the list of results (raises on error)."""
    sh = _Shared(size)
    out = [None] * size
    errs = []

    def body(rank):
        try:
            torch.cuda.set_device(0)
            with torch.cuda.stream(torch.cuda.Stream()):
                out[rank] = fn(ThreadComm(sh, rank))
                torch.cuda.current_stream().synchronize()
        except BaseException as exc:  # noqa: BLE001
            errs.append(exc)
            sh.barrier.abort()

    threads = [threading.Thread(target=body, args=(r,)) for r in range(size)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errs:
        raise errs[0]
    return out
