#!/usr/bin/env python3
"""How fast the generic kernel runs a layout program: `transposeCopy`
(M |> transpose |> map(map(v * 1))) at 8192², timed like the bench's
HBM-bound configs (input sets round robin, steps back to back)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

SRC = ("depFun((n: Nat, m: Nat) => fun(M: Array[n, Array[m, f32]] => "
       "M |> transpose |> mapGlobal(mapGlobal(fun(v => v * 1.0f)))))")


def main():
    import torch
    from paper_2201_03611_b200 import compile_program, emit_cuda
    from paper_2201_03611_b200.run import Executable

    n = m = 8192
    c = compile_program(SRC, None, name="transposeCopy")
    exe = Executable(emit_cuda(c.unit), {"n": n, "m": m})
    print("kernels:", exe.kernel_names, exe.template_kinds)
    sets = [(torch.rand(n * m, device="cuda"), torch.empty(n * m, device="cuda")) for _ in range(2)]
    launches = [exe.bind({"M": a, exe.plan["output"]["name"]: o}) for a, o in sets]
    for i in range(4):
        launches[i % 2]()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(20):
        launches[i % 2]()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    ok = torch.equal(sets[1][1].view(m, n), sets[1][0].view(n, m).t())
    print(f"transposeCopy 8192^2: {ms * 1e3:.1f} us, {8 * n * m / ms / 1e6:.0f} GB/s, exact={ok}")


if __name__ == "__main__":
    main()
