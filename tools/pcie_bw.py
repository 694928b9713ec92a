"""Probe: pinned host <-> device copy bandwidth (1 GiB each way, then both at once on two
streams) — the ceiling of the e2e number."""
import torch, time
n = 1 << 30
d = torch.empty(n // 4, device="cuda")
h = torch.empty(n // 4, pin_memory=True)
for name, f in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
    f(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5): f()
    torch.cuda.synchronize()
    print(name, 5 * n / (time.perf_counter() - t) / 1e9, "GB/s")
# both directions at once on two streams
h2 = torch.empty(n // 4, pin_memory=True); d2 = torch.empty(n // 4, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
print("bidir total", 10 * n / (time.perf_counter() - t) / 1e9, "GB/s")
