#!/usr/bin/env python
"""HBM ceilings by access mix on this GPU (context for the roofline): a
read-only reduction, a copy and a write-only fill over 4 GiB, best of 20
(CUDA events). python scripts/hbm_probe.py"""
import torch, time
A = torch.randn(1 << 30, device="cuda")  # 4 GiB
B = torch.empty_like(A)
def t(f, n=20):
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    best = 1e9
    for _ in range(n):
        e0.record(); f(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best / 1e3
s = t(lambda: A.sum())
print("read-only (A.sum) GB/s", 4 * 2**30 / s / 1e9)
c = t(lambda: B.copy_(A))
print("copy GB/s (r+w)", 8 * 2**30 / c / 1e9)
o = torch.empty(1 << 27, device="cuda")
w = t(lambda: B.fill_(1.0))
print("write-only (fill) GB/s", 4 * 2**30 / w / 1e9)
