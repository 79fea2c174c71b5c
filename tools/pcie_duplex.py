import torch, time
n = 1 << 30
h1 = torch.empty(n, dtype=torch.uint8, pin_memory=True); h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d1 = torch.empty(n, dtype=torch.uint8, device="cuda"); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter()
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    torch.cuda.synchronize(); t1 = time.perf_counter() - t
    t = time.perf_counter()
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize(); t2 = time.perf_counter() - t
    t = time.perf_counter()
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize(); t3 = time.perf_counter() - t
print(f"H2D {t1*1e3:.1f} ms  D2H {t2*1e3:.1f} ms  both concurrent {t3*1e3:.1f} ms")
