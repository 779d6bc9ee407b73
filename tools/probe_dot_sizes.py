#!/usr/bin/env python3
"""The dot reduce kernel at 2^20..2^26 (run under ncu to read per-launch
durations: the fixed per-launch cost vs the streaming rate)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import torch
    from paper_2201_03611_b200 import emit_cuda, programs
    from paper_2201_03611_b200.run import Executable

    code = emit_cuda(programs.compile_config("dot").unit)
    for lg in range(20, 27):
        n = 1 << lg
        exe = Executable(code, {"n": n})
        a = torch.rand(n, device="cuda")
        b = torch.rand(n, device="cuda")
        for _ in range(2):
            exe(a, b)
        torch.cuda.synchronize()


if __name__ == "__main__":
    main()
