import sys; sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/oracle")
import numpy as np
from paper_2201_03611_b200 import compile_program, emit_cuda, programs, run_cuda
c = compile_program(programs.SGEMM, None, name="sgemm")
code = emit_cuda(c.unit)
t = code.text
i = t.index("rise_gemm::gemm_3xtf32_2sm<"); print(t[i:i+200])
for (n, m, k) in [(256, 256, 32), (256, 256, 64)]:
    rng = np.random.default_rng(1)
    A = rng.uniform(-1, 1, (n, k)).astype(np.float32)
    B = rng.uniform(-1, 1, (k, m)).astype(np.float32)
    C = run_cuda(code, c.unit, {"n": n, "m": m, "k": k}, [A, B], as_numpy=True).reshape(n, m)
    R = A.astype(np.float64) @ B.astype(np.float64)
    print(n, m, k, "max|C|", np.abs(C).max(), "max|R|", np.abs(R).max(), "maxerr", np.abs(C - R).max())
    # which reference matches? try C vs A @ (B reinterpreted)
    for name, R2 in [("A@B", R), ("A@B^T-ish", None)]:
        pass
    nz = np.argwhere(np.abs(C) > 0)
    print("nonzero count", len(nz), nz[:5])
