"""Native staged pageable H2D (xmhd_h2d_staged, csrc/hostio.cpp) on this box.

usage: [XMHD_H2D_THREADS=..] [XMHD_H2D_CHUNK_MB=..] [XMHD_H2D_NT=0|1] probe_h2d_native.py
One configuration per process (the staging area is created once)."""
import ctypes
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2108_13622_b200 import _lib, _ops  # noqa: E402

n = 33554432   # one 2048^2 state vector
a = np.random.default_rng(0).standard_normal(n)
lib = _lib.load()
torch.cuda.synchronize()
best = 1e9
for _ in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    d = _ops.as_device(a)
    torch.cuda.synchronize()
    best = min(best, time.perf_counter() - t0)
assert np.array_equal(d.cpu().numpy(), a)
cfg = {k: os.environ.get(k) for k in ("XMHD_H2D_PY", "XMHD_H2D_THREADS", "XMHD_H2D_CHUNK_MB",
                                      "XMHD_H2D_NT", "XMHD_H2D_SLOTS")}
print({k: v for k, v in cfg.items() if v is not None}, "threads", lib.xmhd_h2d_threads(),
      "cores", len(os.sched_getaffinity(0)), round(a.nbytes / best / 1e9, 2), "GB/s")
