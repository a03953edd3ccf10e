import time, numpy as np, torch
for n in (8*4096*4096, 8*8192*8192):
    t0=time.perf_counter(); a=np.random.default_rng(0).standard_normal(n); t1=time.perf_counter()
    print(n, "fresh", round(t1-t0,3), flush=True)
    del a
    t0=time.perf_counter(); h=torch.empty(n, dtype=torch.float64, pin_memory=True); t1=time.perf_counter()
    np.random.default_rng(0).standard_normal(out=h.numpy()); t2=time.perf_counter()
    d=torch.empty(n, dtype=torch.float64, device="cuda"); torch.cuda.synchronize(); t3=time.perf_counter()
    d.copy_(h, non_blocking=True); torch.cuda.synchronize(); t4=time.perf_counter()
    x=torch.from_numpy(h.numpy()).to("cuda"); torch.cuda.synchronize(); t5=time.perf_counter()
    print(n, "pin alloc", round(t1-t0,3), "fill", round(t2-t1,3), "h2d pinned", round(t4-t3,3), "from_numpy.to", round(t5-t4,3), flush=True)
    a=np.random.default_rng(0).standard_normal(n); t6=time.perf_counter(); y=torch.from_numpy(a).to("cuda"); torch.cuda.synchronize(); t7=time.perf_counter()
    print(n, "pageable h2d", round(t7-t6,3), flush=True)
    del a, h, d, x, y
