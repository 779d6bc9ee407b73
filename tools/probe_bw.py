#!/usr/bin/env python3
"""Bandwidth probe: the dot reduce kernel at several sizes (L2 flushed,
events on the launching stream), beside torch's read-only sum and copy —
separates fixed per-launch cost from streaming rate."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def timeit(fn, flush, reps=20):
    import torch
    s = torch.cuda.current_stream()
    ts = []
    for _ in range(3):
        fn()
    for _ in range(reps):
        flush()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        fn()
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2], ts[0]


def main():
    import torch
    from paper_2201_03611_b200 import emit_cuda, programs
    from paper_2201_03611_b200.run import Executable

    c = programs.compile_config("dot")
    code = emit_cuda(c.unit)
    fl = torch.empty(64 << 20, device="cuda")
    sw = torch.ones(64 << 20, device="cuda")
    sink = torch.empty((), device="cuda")

    def flush():
        fl.zero_()
        torch.sum(sw, dim=0, out=sink)

    for lg in (22, 24, 26, 27):
        n = 1 << lg
        exe = Executable(code, {"n": n})
        a = torch.rand(n, device="cuda")
        b = torch.rand(n, device="cuda")
        out = torch.empty(1, device="cuda")
        bound = exe.bind({"a": a, "b": b, "output": out})
        med, best = timeit(bound, flush)
        byt = 8 * n
        t_sum = timeit(lambda: torch.sum(a, dim=0, out=sink), flush)
        dst = torch.empty_like(a)
        t_cp = timeit(lambda: dst.copy_(a), flush)
        print(f"n=2^{lg}: dot {med*1e3:.1f} us ({byt/med/1e6:.0f} GB/s, best {byt/best/1e6:.0f}); "
              f"torch.sum {4*n/t_sum[0]/1e6:.0f} GB/s; copy {8*n/t_cp[0]/1e6:.0f} GB/s", flush=True)
        del exe


if __name__ == "__main__":
    main()
