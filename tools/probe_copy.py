#!/usr/bin/env python3
"""Copy-bandwidth probe at the conv's shape: torch's copy_ of 8192^2 fp32
(256 MiB in, 256 MiB out) over two buffer sets round robin, steps back to
back between two events — the bench's "inputs larger than L2" regime —
beside the conv step in the same regime.  Separates what a read+write
stream of this size reaches from what the stencil reaches."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def rotate_ms(fns, steps=40):
    import torch
    for i in range(6):
        fns[i % len(fns)]()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(steps):
        fns[i % len(fns)]()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def main():
    import torch
    n = 8192 * 8192
    for sets in (2, 3):
        src = [torch.rand(n, device="cuda") for _ in range(sets)]
        dst = [torch.empty(n, device="cuda") for _ in range(sets)]
        fns = [(lambda s=s, d=d: d.copy_(s)) for s, d in zip(src, dst)]
        ms = rotate_ms(fns)
        print(f"torch copy_ 256 MiB -> 256 MiB, {sets} sets: {ms * 1e3:.1f} us, {2 * 4 * n / ms / 1e6:.0f} GB/s")
        fns = [(lambda s=s: torch.sum(s)) for s in src]
        ms = rotate_ms(fns)
        print(f"torch sum 256 MiB, {sets} sets: {ms * 1e3:.1f} us, {4 * n / ms / 1e6:.0f} GB/s")
        del src, dst
    half = n // 2
    src = [torch.rand(half, device="cuda") for _ in range(4)]
    dst = [torch.empty(half, device="cuda") for _ in range(4)]
    fns = [(lambda s=s, d=d: d.copy_(s)) for s, d in zip(src, dst)]
    ms = rotate_ms(fns)
    print(f"torch copy_ 128 MiB -> 128 MiB, 4 sets: {ms * 1e3:.1f} us, {2 * 4 * half / ms / 1e6:.0f} GB/s")


if __name__ == "__main__":
    main()
