#!/usr/bin/env python3
"""Does the relative placement of two input streams matter (HBM channel
alignment)?  The chunked dot (rowfold + seqfold) and the plain dot (reduce)
with b placed at several byte offsets from a 2 MiB-aligned allocation, two
input sets round robin, steps back to back."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import torch
    from paper_2201_03611_b200 import compile_program, emit_cuda, gpu_rules, programs
    from paper_2201_03611_b200.run import Executable

    n = 1 << 24
    stream = torch.cuda.Stream()
    cases = [("dot_chunked", compile_program(programs.DOT, gpu_rules.CHUNKED_REDUCE_STRATEGY, name="dotChunked"),
              {"reassociate": False}),
             ("dot", programs.compile_config("dot"), {})]
    for label, c, kw in cases:
        exe = Executable(emit_cuda(c.unit, **kw), {"n": n})
        for off in (0, 256, 1024, 4096, 65536 + 4096):
            sets = []
            for _ in range(3):
                a = torch.rand(n, device="cuda")
                big = torch.rand(n + off // 4, device="cuda")
                b = big[off // 4:]
                out = torch.empty(exe.output_size, device="cuda")
                bufs = {"a": a, "b": b, "output": out}
                sets.append((exe.graph(bufs, stream) if len(exe.kernels) > 1 else exe.bind(bufs, stream),
                             a, big, out))
            for i in range(6):
                sets[i % 3][0]()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for i in range(30):
                sets[i % 3][0]()
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 30
            print(f"{label} b offset {off:6d} B: {ms * 1e3:.1f} us, {8 * n / ms / 1e6:.0f} GB/s", flush=True)


if __name__ == "__main__":
    main()
