"""The `gridseq` template: a top-level sequential loop enclosing parallel
loops runs over the whole GPU (cooperative grid, grid-wide barriers, grid-
level allocations in global workspaces) instead of one block — bit-exact
with the program's order, the single-block kernel kept for small loops."""

import numpy as np
import pytest

import fast_eval
from paper_2201_03611_b200 import compile_program, emit_cuda, runtime

ROWS_SEQ = ("depFun((n: Nat, m: Nat) => fun(M: Array[n, Array[m, f32]] => "
            "M |> mapSeq(fun(row => row |> mapGlobal(fun(v => v * 2.0f))))))")
# per row: a parallel map into Local memory, then its sequential sum
SEQ_OF_PAR = ("depFun((n: Nat, m: Nat) => fun(M: Array[n, Array[m, f32]] => M |> mapSeq(fun(row => "
              "row |> mapGlobal(fun(v => v * 2.0f)) |> toMem(Local) |> reduceSeq(Private)(fun(a, v => a + v))(0.0f)))))")


@pytest.mark.parametrize("src,name", [(ROWS_SEQ, "rowsSeq"), (SEQ_OF_PAR, "seqOfPar")])
def test_gridseq_selected_with_the_single_block_fallback(src, name):
    c = compile_program(src, None, name=name)
    code = emit_cuda(c.unit)
    (st,) = code.plan["stages"]
    assert st["kind"] == "gridseq" and st["cooperative"] and st["fallback"]["kind"] == "block"
    assert st["pre"] == ["(m) >= 4096"]
    names = [f"{st['name']}<4, 8192>", f"{st['fallback']['name']}<4, 8192>"]
    cubin, _ = runtime.compile_cubin(code.text, names, ["--fmad=false"])
    assert cubin[:4] == b"\x7fELF"
    # order-preserving: kept under reassociate=False
    assert emit_cuda(c.unit, reassociate=False).plan["stages"][0]["kind"] == "gridseq"


@pytest.mark.gpu
@pytest.mark.parametrize("src,name", [(ROWS_SEQ, "rowsSeq"), (SEQ_OF_PAR, "seqOfPar")])
@pytest.mark.parametrize("n,m", [(5, 8192), (3, 100000), (4, 100)])
def test_gridseq_bit_exact(gpu, src, name, n, m):
    from paper_2201_03611_b200.run import Executable, run_cuda

    c = compile_program(src, None, name=name)
    code = emit_cuda(c.unit)
    M = np.random.default_rng(7).uniform(-1, 1, (n, m)).astype(np.float32)
    got = run_cuda(code, c.unit, {"n": n, "m": m}, [M], as_numpy=True)
    want = np.asarray(fast_eval.to_numpy(fast_eval.eval_program(c.source_typed, {"n": n, "m": m}, [M])),
                      np.float32).reshape(-1)
    np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32))
    kinds = Executable(code, {"n": n, "m": m}).template_kinds
    assert kinds == (["gridseq"] if m >= 4096 else ["block"])
