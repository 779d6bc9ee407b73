#!/usr/bin/env python3
"""How fast layout programs run (transpose, slide,
padClamp, split/join) — each at ≈ 2^26 elements, timed like the bench's
HBM-bound configs (two input sets round robin, steps back to back), with
the template (or generic kernel) that took it and the bytes it must move."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

N2 = 8192
N1 = 1 << 26
PROGRAMS = [
    ("transposeCopy", "depFun((n: Nat, m: Nat) => fun(M: Array[n, Array[m, f32]] => "
                      "M |> transpose |> mapGlobal(mapGlobal(fun(v => v * 1.0f)))))",
     {"n": N2, "m": N2}, [N2 * N2], N2 * N2),
    ("pad2DCopy", "depFun((n: Nat, m: Nat) => fun(M: Array[n, Array[m, f32]] => M |> padClamp2D(1)(2) "
                  "|> mapGlobal(mapGlobal(fun(v => v * 1.0f)))))",
     {"n": N2, "m": N2}, [N2 * N2], (N2 + 3) * (N2 + 3)),
    ("slide1D", "depFun((n: Nat) => fun(xs: Array[n, f32] => xs |> padClamp(1)(1) |> slide(3)(1) "
                "|> mapGlobal(fun(w => w |> reduceSeq(Private)(fun(a, v => a + v))(0.0f)))))",
     {"n": N1}, [N1], N1),
    ("splitJoinScale", "depFun((n: Nat) => fun(xs: Array[4 * n, f32] => xs |> split(4) "
                       "|> mapGlobal(fun(c => c |> mapSeq(fun(v => v * 0.5f)))) |> join))",
     {"n": N1 // 4}, [N1], N1),
]


def main():
    import torch
    from paper_2201_03611_b200 import compile_program, emit_cuda
    from paper_2201_03611_b200.run import Executable

    for name, src, nats, in_sizes, out_size in PROGRAMS:
        c = compile_program(src, None, name=name)
        exe = Executable(emit_cuda(c.unit), nats)
        in_names = [i["name"] for i in exe.plan["inputs"]]
        sets = []
        for _ in range(2):
            bufs = {nm: torch.rand(sz, device="cuda") for nm, sz in zip(in_names, in_sizes)}
            bufs[exe.plan["output"]["name"]] = torch.empty(exe.output_size, device="cuda")
            sets.append(exe.bind(bufs))
        for i in range(4):
            sets[i % 2]()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(20):
            sets[i % 2]()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        nbytes = 4 * (sum(in_sizes) + out_size)
        print(f"{name}: {exe.template_kinds} {ms * 1e3:.1f} us, {nbytes / ms / 1e6:.0f} GB/s", flush=True)


if __name__ == "__main__":
    main()
