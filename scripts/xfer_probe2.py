import time, numpy as np, torch, threading
n = 16384
d = torch.rand((n, n), dtype=torch.float64, device="cuda")
C = np.random.default_rng(0).random((n, n))
torch.cuda.synchronize()
def t(f, label, nb=d.numel()*8):
    torch.cuda.synchronize(); t0 = time.perf_counter(); r = f(); torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"{label}: {dt*1e3:.1f} ms  {nb/dt/1e9:.1f} GB/s", flush=True); return r
t(lambda: torch.empty(n * n, dtype=torch.float64).pin_memory(), "alloc+pin 2GB via pin_memory()")
t(lambda: torch.empty(n * n, dtype=torch.float64, pin_memory=True), "torch.empty(pin_memory=True) 2GB")
pinned = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
t(lambda: pinned.copy_(d), "D2H into pinned")
def threaded(dst_np, src, nthreads, h2d=False):
    rows = np.array_split(np.arange(n), nthreads)
    def work(r):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            if h2d:
                src[r[0]:r[-1]+1].copy_(torch.from_numpy(dst_np[r[0]:r[-1]+1]))
            else:
                torch.from_numpy(dst_np[r[0]:r[-1]+1]).copy_(src[r[0]:r[-1]+1])
        s.synchronize()
    ths = [threading.Thread(target=work, args=(r,)) for r in rows]
    [x.start() for x in ths]; [x.join() for x in ths]
for nt in (4, 8, 16):
    out = np.empty((n, n))
    t(lambda: threaded(out, d, nt), f"D2H pageable fresh, {nt} threads")
    t(lambda: threaded(C, d, nt, h2d=True), f"H2D pageable, {nt} threads")
out = np.empty((n, n))
def touch(a, nt=16):
    parts = np.array_split(np.arange(a.shape[0]), nt)
    ths = [threading.Thread(target=lambda r=r: a[r[0]:r[-1]+1].fill(0.0)) for r in parts]
    [x.start() for x in ths]; [x.join() for x in ths]
t(lambda: touch(out), "parallel first-touch 2GB (16 threads)")
t(lambda: torch.from_numpy(out).copy_(d), "D2H pageable pre-touched")
