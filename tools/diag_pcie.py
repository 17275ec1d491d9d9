"""PCIe copy rates of this box (diagnostic): H2D, D2H alone and concurrently."""
import time
import torch
n = 64 << 20
h1, h2 = torch.empty(n, dtype=torch.uint8).pin_memory(), torch.empty(n, dtype=torch.uint8).pin_memory()
d1, d2 = torch.empty(n, dtype=torch.uint8, device="cuda"), torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for name, fn in (("h2d", lambda: d1.copy_(h1, non_blocking=True)), ("d2h", lambda: h2.copy_(d2, non_blocking=True))):
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(10): fn()
    torch.cuda.synchronize(); print(name, n * 10 / (time.perf_counter() - t) / 1e9, "GB/s")
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(10):
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t
print("both", 2 * n * 10 / dt / 1e9, "GB/s aggregate")
