"""PCIe probe: one pinned 4.29 GB block host -> device and back, as one copy,
as 8 slab copies on one stream, and as slabs spread over 2 / 4 streams."""
import time, torch
n = 2048 * 2048 * 128
h = torch.empty(n, dtype=torch.float64).pin_memory()
h.uniform_(-1, 1)
d = torch.empty(n, dtype=torch.float64, device="cuda")
h2 = torch.empty(n, dtype=torch.float64).pin_memory()

def run(direction, nstream, nslab):
    streams = [torch.cuda.Stream() for _ in range(nstream)]
    step = n // nslab
    best = 1e9
    for _ in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for s in range(nslab):
            a, e = s * step, (s + 1) * step
            with torch.cuda.stream(streams[s % nstream]):
                if direction == "h2d":
                    d[a:e].copy_(h[a:e], non_blocking=True)
                else:
                    h2[a:e].copy_(d[a:e], non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best

for direction in ("h2d", "d2h"):
    for nstream, nslab in ((1, 1), (1, 8), (2, 8), (4, 8), (2, 2), (4, 32)):
        t = run(direction, nstream, nslab)
        print(f"{direction} streams {nstream} slabs {nslab}: {t*1e3:.2f} ms, {n*8/t/1e9:.1f} GB/s")
assert torch.equal(h, h2)
# both directions at once (full duplex)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
torch.cuda.synchronize(); t0 = time.perf_counter()
with torch.cuda.stream(s1): d2.copy_(h, non_blocking=True)
with torch.cuda.stream(s2): h2.copy_(d, non_blocking=True)
torch.cuda.synchronize(); t = time.perf_counter() - t0
print(f"duplex: {t*1e3:.2f} ms, {n*8/t/1e9:.1f} GB/s each way")
