import time, ctypes, numpy as np, torch, threading
n = 16384
C = np.random.default_rng(0).random((n, n))
d = torch.empty((n, n), dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
def t(f, label):
    torch.cuda.synchronize(); t0 = time.perf_counter(); f(); torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"{label}: {dt*1e3:.1f} ms  {C.nbytes/dt/1e9:.1f} GB/s", flush=True)
t(lambda: d.copy_(torch.from_numpy(C)), "pageable copy_ H2D")
t(lambda: d.copy_(torch.from_numpy(C)), "pageable copy_ H2D (2nd)")
out = np.empty_like(C)
t(lambda: torch.from_numpy(out).copy_(d), "pageable D2H")
cr = torch.cuda.cudart()
def reg():
    r = cr.cudaHostRegister(C.ctypes.data, C.nbytes, 0); assert r == 0, r
t(reg, "cudaHostRegister 2 GB")
t(lambda: d.copy_(torch.from_numpy(C), non_blocking=True), "registered H2D")
t(lambda: cr.cudaHostUnregister(C.ctypes.data), "unregister")
# pinned staging with threads
CH = 64 << 20
bufs = [torch.empty(CH // 8, dtype=torch.float64).pin_memory() for _ in range(4)]
flat_d = d.view(-1)
flat = C.reshape(-1)
s = torch.cuda.Stream()
def staged(nthreads=8):
    evs = [None] * 4
    nchunks = (flat.size * 8 + CH - 1) // CH
    for k in range(nchunks):
        b = k % 4
        if evs[b] is not None: evs[b].synchronize()
        lo = k * (CH // 8); hi = min(flat.size, lo + CH // 8)
        dst = bufs[b].numpy()[: hi - lo]
        parts = np.array_split(np.arange(lo, hi), nthreads)
        ths = [threading.Thread(target=lambda a=a: np.copyto(dst[a[0]-lo:a[-1]-lo+1], flat[a[0]:a[-1]+1])) for a in parts if len(a)]
        [x.start() for x in ths]; [x.join() for x in ths]
        with torch.cuda.stream(s):
            flat_d[lo:hi].copy_(bufs[b][: hi - lo], non_blocking=True)
            evs[b] = torch.cuda.Event(); evs[b].record(s)
    s.synchronize()
t(staged, "pinned staging 8 threads H2D")
