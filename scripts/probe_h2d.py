"""Pageable NumPy -> device copy paths on this box (e2e's H2D): plain
torch.from_numpy(a).cuda(), a staged pipeline through page-locked chunks
filled by host threads, and cudaHostRegister of the caller's buffer."""
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

n = 33554432
a = np.random.default_rng(0).standard_normal(n)
dev = torch.empty(n, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()


def t(f, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return a.nbytes / best / 1e9


print("plain .cuda()", round(t(lambda: dev.copy_(torch.from_numpy(a))), 2), "GB/s")
for chunk_mb, threads in ((8, 4), (16, 8), (32, 8), (16, 16)):
    chunk = chunk_mb * (1 << 20) // 8
    nslot = 4
    slots = [torch.empty(chunk, dtype=torch.float64, pin_memory=True) for _ in range(nslot)]
    evs = [None] * nslot
    pool = ThreadPoolExecutor(threads)
    side = torch.cuda.Stream()

    def staged():
        k = 0
        for i0 in range(0, n, chunk):
            m = min(chunk, n - i0)
            s = k % nslot
            if evs[s] is not None:
                evs[s].synchronize()
            buf = slots[s].numpy()
            parts = np.linspace(0, m, threads + 1).astype(int)
            list(pool.map(lambda j: np.copyto(buf[parts[j]:parts[j + 1]],
                                              a[i0 + parts[j]:i0 + parts[j + 1]]), range(threads)))
            with torch.cuda.stream(side):
                dev[i0:i0 + m].copy_(slots[s][:m], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(side)
            evs[s] = ev
            k += 1
        side.synchronize()

    print(f"staged {chunk_mb} MB x {threads} threads", round(t(staged), 2), "GB/s")

cr = torch.cuda.cudart()


def registered():
    ptr = a.ctypes.data
    cr.cudaHostRegister(ptr, a.nbytes, 0)
    dev.copy_(torch.from_numpy(a), non_blocking=True)
    torch.cuda.synchronize()
    cr.cudaHostUnregister(ptr)


print("cudaHostRegister + copy + unregister", round(t(registered), 2), "GB/s")
host = torch.empty(n, dtype=torch.float64, pin_memory=True)
print("pinned -> device", round(t(lambda: dev.copy_(host, non_blocking=True)), 2), "GB/s")
print("device -> pinned", round(t(lambda: host.copy_(dev, non_blocking=True)), 2), "GB/s")
print("device -> pageable", round(t(lambda: dev.cpu()), 2), "GB/s")
