import time, torch
n = 1 << 27
h1 = torch.empty(n, dtype=torch.float64).pin_memory(); h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d1 = torch.empty(n, dtype=torch.float64, device="cuda"); d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=5):
    fn(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps
gb = n * 8 / 1e9
h2d = t(lambda: d1.copy_(h1, non_blocking=True)); d2h = t(lambda: h2.copy_(d2, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
bo = t(both)
print(f"H2D {gb/h2d:.1f} GB/s  D2H {gb/d2h:.1f} GB/s  both concurrently {2*gb/bo:.1f} GB/s total ({bo*1e3:.1f} ms for 2x{gb:.2f} GB)")
