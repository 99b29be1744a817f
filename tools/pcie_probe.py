"""PCIe ceiling on this box: pinned H2D alone, D2H alone, both at once."""
import time

import torch

n = 64 * 1024 * 1024  # 256 MB
h1 = torch.empty(n).pin_memory()
h2 = torch.empty(n).pin_memory()
d1 = torch.empty(n, device="cuda")
d2 = torch.empty(n, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    d1.copy_(h1, non_blocking=True)
    h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
def run(h2d, d2h, reps=5):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s1):
                d1.copy_(h1, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps
for name, a, b in (("H2D", 1, 0), ("D2H", 0, 1), ("both", 1, 1)):
    t = run(a, b)
    print(f"{name}: {4 * n / t / 1e9:.1f} GB/s per direction")
