"""SURVEY.md §8 f 4: vector types and memory reuse.

* `asVector(w)` / `asScalar` (extension primitives: split / join as values,
  w-aligned contiguous vectors as memory accesses) through every seam —
  typing, DPIA, lowering, `eval_program`, `run_unit`, the reference's own C
  emitter, the vectorised oracle — and float4 / float2 loads and stores in
  the sm100a generic kernel, with the scalar kernel as the fallback for
  unaligned buffers;
* reuse of Global temporaries (toMem(Global)) whose stage lifetimes do not
  overlap."""

import random

import numpy as np
import pytest

import fast_eval
from paper_2201_03611_b200 import compile_program, emit_cuda, runtime
from paper_2201_03611_b200._ref import cexec, codegen, interpreter, nat

SAXPY4 = """depFun((n: Nat) => fun(xs: Array[n, f32] => fun(ys: Array[n, f32] =>
  zip(xs |> asVector(4))(ys |> asVector(4))
    |> mapGlobal(fun(p => zip(fst(p))(snd(p)) |> mapSeq(fun(q => fst(q) * 2.0f + snd(q)))))
    |> asScalar)))"""

# a vector-wise row sum: each work-item folds its float2 lanes of a row
ROWS2 = """depFun((n: Nat, m: Nat) => fun(M: Array[n, Array[m, f32]] =>
  M |> mapGlobal(fun(row => row |> asVector(2)
      |> reduceSeq(Private)(fun(acc, v => acc + (v |> reduceSeq(Private)(fun(a, x => a + x))(0.0f))))(0.0f) ))))"""

CHAIN = """depFun((n: Nat) => fun(xs: Array[n, f32] =>
  xs |> mapGlobal(fun(x => x * 2.0f)) |> toMem(Global) |> mapGlobal(fun(x => x + 1.0f)) |> toMem(Global)
     |> mapGlobal(fun(x => x * 3.0f)) |> toMem(Global) |> mapGlobal(fun(x => x - 1.0f))))"""


def _saxpy():
    return compile_program(SAXPY4, None, name="saxpy4", assumptions=[(nat.Var("n"), nat.Const(4))])


def _inputs(n, seed=3):
    rng = np.random.default_rng(seed)
    return [rng.uniform(-1, 1, n).astype(np.float32), rng.uniform(-1, 1, n).astype(np.float32)]


def test_as_vector_values_are_split_and_join():
    c = _saxpy()
    xs, ys = _inputs(12)
    want = interpreter.to_plain(interpreter.eval_program(c.source_typed, {"n": 12}, [list(xs), list(ys)]))
    fast = fast_eval.to_numpy(fast_eval.eval_program(c.source_typed, {"n": 12}, [xs, ys]))
    ref = (xs * np.float32(2.0) + ys).astype(np.float32)
    np.testing.assert_array_equal(np.asarray(want, np.float32), ref)
    np.testing.assert_array_equal(np.asarray(fast, np.float32), ref)
    # the imperative oracle through the acceptor duals (asScalarAcc)
    got = interpreter.run_unit(c.unit, {"n": 12}, [list(xs), list(ys)])
    np.testing.assert_array_equal(np.asarray(interpreter.to_plain(got), np.float32), ref)


def test_reference_c_emitter_handles_the_vector_views():
    c = _saxpy()
    code = codegen.emit(c.unit, "opencl")
    xs, ys = _inputs(8)
    got = cexec.run_emitted(code, c.unit, {"n": 8}, [list(xs), list(ys)])
    np.testing.assert_array_equal(np.asarray(got, np.float32), (xs * np.float32(2) + ys).astype(np.float32))


def test_sm100a_emits_float4_accesses_with_a_scalar_fallback():
    code = emit_cuda(_saxpy().unit)
    (st,) = code.plan["stages"]
    assert st.get("vector") and st["name"].endswith("_vec") and st["fallback"]["kind"] == "grid"
    body = code.text[code.text.index(st["name"] + "("):]
    assert body.count("*reinterpret_cast<const float4*>") == 2 and "*reinterpret_cast<float4*>(output" in body
    names = [f"{st['name']}<4096>", f"{st['fallback']['name']}<4096>"]
    cubin, lowered = runtime.compile_cubin(code.text, names, ["--fmad=false"])
    assert cubin[:4] == b"\x7fELF"


def test_float2_lanes_inside_a_fold():
    c = compile_program(ROWS2, None, name="rows2", assumptions=[(nat.Var("m"), nat.Const(2))])
    code = emit_cuda(c.unit, idioms=False)
    st = code.plan["stages"][0]
    assert st.get("vector") and "reinterpret_cast<const float2*>" in code.text


def test_unaligned_vectors_stay_scalar():
    # a vector view over a transposed matrix is not contiguous: no vector access
    src = """depFun((n: Nat, m: Nat) => fun(M: Array[n, Array[m, f32]] =>
      M |> transpose |> mapGlobal(fun(col => col |> asVector(4)
          |> mapSeq(fun(v => v |> reduceSeq(Private)(fun(a, x => a + x))(0.0f))) )) ))"""
    c = compile_program(src, None, name="colsum", assumptions=[(nat.Var("n"), nat.Const(4))])
    code = emit_cuda(c.unit, idioms=False)
    assert not any(s.get("vector") for s in code.plan["stages"])


def test_global_temporaries_reuse_slots():
    c = compile_program(CHAIN, None, name="chain")
    temps = emit_cuda(c.unit).plan["temps"]
    slots = {t["name"]: t["slot"] for t in temps}
    # tmp (stages 0-1) and tmp2 (stages 2-3) never live at once; tmp1 overlaps both
    assert len(temps) == 3 and len(set(slots.values())) == 2
    assert slots[temps[0]["name"]] == slots[temps[2]["name"]] != slots[temps[1]["name"]]


@pytest.mark.gpu
@pytest.mark.parametrize("n", [4, 4096, 1 << 22])
def test_vector_kernel_bit_exact_and_fallback_for_unaligned(gpu, n):
    import torch

    from paper_2201_03611_b200 import run_cuda
    from paper_2201_03611_b200.run import Executable

    c = _saxpy()
    code = emit_cuda(c.unit)
    xs, ys = _inputs(n)
    want = (xs * np.float32(2) + ys).astype(np.float32)
    got = run_cuda(code, c.unit, {"n": n}, [xs, ys], as_numpy=True)
    np.testing.assert_array_equal(got, want)
    exe = Executable(code, {"n": n})
    assert exe.kernel_names == ["saxpy4Kernel_vec"]
    big = torch.zeros(n + 1, dtype=torch.float32, device="cuda")
    big[1:] = torch.from_numpy(xs).cuda()
    out = exe(big[1:], torch.from_numpy(ys).cuda())  # 4-byte offset: the scalar kernel runs
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out.cpu().numpy(), want)


@pytest.mark.gpu
def test_float2_fold_and_reused_temporaries_on_the_gpu(gpu):
    from paper_2201_03611_b200 import run_cuda

    c = compile_program(ROWS2, None, name="rows2", assumptions=[(nat.Var("m"), nat.Const(2))])
    M = np.random.default_rng(4).uniform(-1, 1, (33, 64)).astype(np.float32)
    got = run_cuda(emit_cuda(c.unit), c.unit, {"n": 33, "m": 64}, [M], as_numpy=True)
    want = fast_eval.to_numpy(fast_eval.eval_program(c.source_typed, {"n": 33, "m": 64}, [M]))
    np.testing.assert_array_equal(got, np.asarray(want, np.float32))
    c = compile_program(CHAIN, None, name="chain")
    xs = _inputs(1 << 20)[0]
    got = run_cuda(emit_cuda(c.unit), c.unit, {"n": 1 << 20}, [xs], as_numpy=True)
    x = (xs * np.float32(2)).astype(np.float32)
    x = (x + np.float32(1)).astype(np.float32)
    x = (x * np.float32(3)).astype(np.float32)
    np.testing.assert_array_equal(got, (x - np.float32(1)).astype(np.float32))
