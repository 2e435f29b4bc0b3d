"""Host-side copy costs behind the end-to-end number: pinned D2H bandwidth,
first-touch cost of fresh numpy buffers, pinned->pageable memcpy."""
import time

import numpy as np
import torch

n = 420 << 20
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d.fill_(1)
p = torch.empty(n, dtype=torch.uint8, pin_memory=True)
for _ in range(2):
    torch.cuda.synchronize()
    t = time.perf_counter()
    p.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
print(f"D2H pinned {n / dt / 1e9:.1f} GB/s ({dt * 1e3:.1f} ms for {n >> 20} MB)")
for _ in range(2):
    t = time.perf_counter()
    a = np.empty(n, dtype=np.uint8)
    a[::4096] = 0  # first touch of every page
    dt = time.perf_counter() - t
print(f"first touch of a fresh {n >> 20} MB numpy buffer: {dt * 1e3:.1f} ms")
src = p.numpy()
t = time.perf_counter()
b = np.empty(n, dtype=np.uint8)
np.copyto(b, src)
dt = time.perf_counter() - t
print(f"pinned -> fresh numpy memcpy (1 thread): {n / dt / 1e9:.1f} GB/s")
t = time.perf_counter()
np.copyto(b, src)
dt = time.perf_counter() - t
print(f"pinned -> touched numpy memcpy (1 thread): {n / dt / 1e9:.1f} GB/s")
print(open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip())
