"""Host<->device copy bandwidth from pinned memory: one copy vs chunks on several streams."""
import time

import torch

n = 268435456 // 8
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


streams = [torch.cuda.Stream() for _ in range(4)]


def chunked(direction, k):
    def fn():
        cur = torch.cuda.current_stream()
        step = (n + k - 1) // k
        for i in range(k):
            s = streams[i % len(streams)]
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                a, b = i * step, min(n, (i + 1) * step)
                if direction == "h2d":
                    d[a:b].copy_(h[a:b], non_blocking=True)
                else:
                    h[a:b].copy_(d[a:b], non_blocking=True)
        for s in streams:
            cur.wait_stream(s)
    return fn


for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)),
                 ("d2h", lambda: h.copy_(d, non_blocking=True))):
    dt = timed(fn)
    print(name, f"single {dt*1e3:.2f} ms  {n*8/dt/1e9:.1f} GB/s", flush=True)
for direction in ("h2d", "d2h"):
    for k in (2, 4, 8):
        dt = timed(chunked(direction, k))
        print(direction, f"chunks={k} {dt*1e3:.2f} ms  {n*8/dt/1e9:.1f} GB/s", flush=True)
