#!/usr/bin/env python3
"""PCIe duplex: H2D alone, D2H alone, and both at once on two streams (the
conv e2e's overlap of step k+1's upload with step k-1's download).  Probe only."""
import torch

n = 268435456 // 4
h_in = torch.empty(n).pin_memory()
h_out = torch.empty(n).pin_memory()
d_in = torch.empty(n, device="cuda")
d_out = torch.empty(n, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(f, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


print("H2D alone", round(268.4 / t(lambda: d_in.copy_(h_in, non_blocking=True)), 1), "GB/s")
print("D2H alone", round(268.4 / t(lambda: h_out.copy_(d_out, non_blocking=True)), 1), "GB/s")
ms = t(both)
print("both at once", round(2 * 268.4 / ms, 1), "GB/s total,", round(268.4 / ms, 1), "each")
