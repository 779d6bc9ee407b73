#!/usr/bin/env python3
"""Accuracy + timing of one gemm_tc variant (env RISE_GEMM_*), for sweeps."""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))


def main():
    import torch

    import oracle
    from paper_2201_03611_b200 import compile_program, emit_cuda, programs, run_cuda
    from paper_2201_03611_b200.run import Executable

    c = compile_program(programs.SGEMM_BT, None, name="sgemm")
    code = emit_cuda(c.unit)
    n = 1024
    A = oracle.rng_inputs(4, n, n)
    Bt = oracle.rng_inputs(14, n, n)
    got = run_cuda(code, c.unit, {"n": n, "m": n, "k": n}, [A, Bt], as_numpy=True).reshape(n, n)
    C64, absC = oracle.sgemm_bt_f64(A[:128], Bt)
    rel = float(np.max(np.abs(got[:128] - C64) / absC))
    N = 4096
    exe = Executable(code, {"n": N, "m": N, "k": N})
    a = torch.rand(N * N, device="cuda") - 0.5
    b = torch.rand(N * N, device="cuda") - 0.5
    out = torch.empty(N * N, device="cuda")
    for _ in range(3):
        exe(a, b, out=out)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        exe(a, b, out=out)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(json.dumps({"variant": code.plan["stages"][0]["name"], "plan_bn": code.plan["stages"][0].get("bn"),
                      "max_rel_err_vs_sum_abs": rel, "best_ms": best, "tflops": 2 * N ** 3 / best / 1e9}))


if __name__ == "__main__":
    main()
