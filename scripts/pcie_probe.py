import time, numpy as np, torch

a = np.ones((40000, 20, 20), dtype=np.int8)
rt = torch.cuda.cudart()
print("register rc", int(rt.cudaHostRegister(a.ctypes.data, a.nbytes, 0)))
d = torch.empty(a.shape, dtype=torch.int8, device="cuda")
t = torch.from_numpy(a)
print("is_pinned", t.is_pinned())
for name, fn in (("h2d", lambda: d.copy_(t, non_blocking=True)), ("d2h", lambda: t.copy_(d, non_blocking=True))):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20): fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 20
    print(name, "%.1f us  %.1f GB/s" % (dt * 1e6, a.nbytes / dt / 1e9))
p = torch.empty(a.shape, dtype=torch.int8).pin_memory()
for name, fn in (("h2d_pinned", lambda: d.copy_(p, non_blocking=True)), ("d2h_pinned", lambda: p.copy_(d, non_blocking=True))):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20): fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 20
    print(name, "%.1f us  %.1f GB/s" % (dt * 1e6, a.nbytes / dt / 1e9))
s2 = torch.cuda.Stream()
t0 = time.perf_counter()
for _ in range(20):
    d.copy_(p, non_blocking=True)
    with torch.cuda.stream(s2):
        p.copy_(d, non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / 20
print("bidir", "%.1f us" % (dt * 1e6))
