import torch, time
n = 1 << 28  # 1 GiB in bytes (uint8)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
h = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
for name, fn in (("D2H", lambda: h.copy_(d, non_blocking=True)), ("H2D", lambda: d.copy_(h, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); [fn() for _ in range(5)]; e1.record(); torch.cuda.synchronize()
    print(name, 5 * n / (e0.elapsed_time(e1) / 1e3) / 1e9, "GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(s1): h.copy_(d, non_blocking=True)
    with torch.cuda.stream(s2): d2.copy_(h2, non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t0
print("duplex", 2 * 5 * n / dt / 1e9, "GB/s total")
# chunked D2H of 1.5 MB pieces
m = 1500000
torch.cuda.synchronize(); t0 = time.perf_counter()
for k in range(0, n - m, m):
    h[k:k+m].copy_(d[k:k+m], non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t0
print("chunked 1.5MB D2H", n / dt / 1e9, "GB/s")
