"""Pinned host <-> device copy bandwidth: H2D, D2H and both at once (two streams)."""
import time

import torch

n = 512 << 20
h1 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for name, fn in (("h2d", lambda: d1.copy_(h1, non_blocking=True)),
                 ("d2h", lambda: h2.copy_(d2, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    print(name, f"{5 * n / (time.perf_counter() - t) / 1e9:.1f} GB/s")
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
print("both", f"{10 * n / (time.perf_counter() - t) / 1e9:.1f} GB/s aggregate")
