"""Layout and extension-primitive programs on the GPU (north star: bit-exact
for index/layout patterns — split/join/transpose/slide/pad — and for any
program whose order the kernel keeps).  The oracle is the reference's
imperative interpreter `run_unit` with the extension semantics
(extension.py §4), compared BIT FOR BIT (not within 4 ULP), plus numpy
restatements at sizes the interpreter would take minutes on."""

import random

import numpy as np
import pytest

from paper_2201_03611_b200 import compile_program, emit_cuda, run_cuda
from paper_2201_03611_b200._ref import interpreter

pytestmark = pytest.mark.gpu

CONV5 = """depFun((n: Nat, m: Nat) => fun(img: Array[n, Array[m, f32]] => fun(w: Array[5, Array[5, f32]] =>
  img |> padClamp2D(2)(2) |> slide2D(5)(1) |> mapGlobal(mapGlobal(fun(win =>
    zip(win)(w)
      |> mapSeq(fun(rw => zip(fst(rw))(snd(rw)) |> reduceSeq(Private)(fun(acc, p => acc + fst(p) * snd(p)))(0.0f)))
      |> toMem(Private)
      |> reduceSeq(Private)(fun(acc, v => acc + v))(0.0f) ))) )))"""

PROGRAMS = {
    "transposeCopy": ("depFun((n: Nat, m: Nat) => fun(M: Array[n, Array[m, f32]] => "
                      "M |> transpose |> mapGlobal(mapGlobal(fun(v => v * 1.0f)))))", {"n": 5, "m": 7}),
    "slide1D": ("depFun((n: Nat) => fun(xs: Array[n, f32] => xs |> padClamp(1)(1) |> slide(3)(1) "
                "|> mapGlobal(fun(w => w |> reduceSeq(Private)(fun(a, v => a + v))(0.0f)))))", {"n": 9}),
    "slideStride2": ("depFun((n: Nat) => fun(xs: Array[2 * n + 4, f32] => xs |> slide(4)(2) "
                     "|> mapGlobal(fun(w => w |> reduceSeq(Private)(fun(a, v => a + v))(0.0f)))))", {"n": 6}),
    "splitJoinScale": ("depFun((n: Nat) => fun(xs: Array[4 * n, f32] => xs |> split(4) "
                       "|> mapGlobal(fun(c => c |> mapSeq(fun(v => v * 0.5f)))) |> join))", {"n": 5}),
    "padClampCopy": ("depFun((n: Nat) => fun(xs: Array[n, f32] => xs |> padClamp(2)(3) "
                     "|> mapGlobal(fun(v => v * 1.0f))))", {"n": 6}),
    "pad2DCopy": ("depFun((n: Nat, m: Nat) => fun(M: Array[n, Array[m, f32]] => M |> padClamp2D(1)(2) "
                  "|> mapGlobal(mapGlobal(fun(v => v * 1.0f)))))", {"n": 4, "m": 5}),
    "conv5": (CONV5, {"n": 9, "m": 12}),
    "divSqrt": ("depFun((n: Nat) => fun(a: Array[n, f32] => fun(b: Array[n, f32] => zip(a)(b) |> mapGlobal(fun(p => "
                "div(sqrt(fst(p) * fst(p) + snd(p) * snd(p)))(snd(p) * snd(p) + 1.0f))))))", {"n": 11}),
}


def _value(dtype, nats, rng):
    from paper_2201_03611_b200._ref import nat, types

    if isinstance(dtype, types.ArrayType):
        return [_value(dtype.elem, nats, rng) for _ in range(nat.evaluate(dtype.size, nats))]
    return np.float32(rng.uniform(-4.0, 4.0))


def _bits(v):
    return np.asarray(v, dtype=np.float32).reshape(-1).view(np.uint32)


@pytest.mark.parametrize("name", sorted(PROGRAMS))
def test_program_bit_exact_with_run_unit(gpu, name):
    src, nats = PROGRAMS[name]
    c = compile_program(src, None, name=name)
    code = emit_cuda(c.unit)
    rng = random.Random(sum(map(ord, name)))
    for _ in range(5):
        inputs = [_value(dt, nats, rng) for _v, dt in c.unit.inputs]
        got = run_cuda(code, c.unit, nats, inputs)
        ref = interpreter.run_unit(c.unit, nats, inputs, strict=True)
        np.testing.assert_array_equal(_bits(got), _bits(ref), err_msg=name)


def _run(name, nats, arrays):
    src, _ = PROGRAMS[name]
    c = compile_program(src, None, name=name)
    return c, run_cuda(emit_cuda(c.unit), c.unit, nats, arrays, as_numpy=True)


def test_transpose_and_pads_at_size(gpu):
    rng = np.random.default_rng(7)
    M = rng.standard_normal((300, 517)).astype(np.float32)
    _, got = _run("transposeCopy", {"n": 300, "m": 517}, [M])
    np.testing.assert_array_equal(got.reshape(517, 300), M.T)
    _, got = _run("pad2DCopy", {"n": 300, "m": 517}, [M])
    np.testing.assert_array_equal(got.reshape(303, 520), np.pad(M, ((1, 2), (1, 2)), mode="edge"))
    xs = rng.standard_normal(10001).astype(np.float32)
    _, got = _run("padClampCopy", {"n": 10001}, [xs])
    np.testing.assert_array_equal(got, np.pad(xs, (2, 3), mode="edge"))


def test_slides_at_size(gpu):
    rng = np.random.default_rng(8)
    xs = rng.standard_normal(100003).astype(np.float32)
    _, got = _run("slide1D", {"n": 100003}, [xs])
    p = np.pad(xs, (1, 1), mode="edge")
    want = ((np.float32(0) + p[:-2]) + p[1:-1]) + p[2:]
    np.testing.assert_array_equal(got, want.astype(np.float32))
    n = 5000
    ys = rng.standard_normal(2 * n + 4).astype(np.float32)
    _, got = _run("slideStride2", {"n": n}, [ys])
    idx = 2 * np.arange(n + 1)
    want = np.float32(0)
    for k in range(4):  # left fold over the window, in order
        want = (want + ys[idx + k]).astype(np.float32)
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("n,m", [(9, 12), (70, 136), (257, 520)])
def test_conv5_stencil_template_bit_exact(gpu, n, m):
    """A 5x5 window through the stencil2d template (halo 2, packed exact
    FFMA2/FADD2 body) against a numpy restatement of the program's order:
    each window row folded left from 0.0f, then the row sums folded."""
    rng = np.random.default_rng(n * m)
    img = rng.uniform(-1, 1, (n, m)).astype(np.float32)
    w = rng.uniform(-1, 1, (5, 5)).astype(np.float32)
    c, got = _run("conv5", {"n": n, "m": m}, [img, w])
    if m % 4 == 0:
        assert emit_cuda(c.unit).plan["stages"][0]["kind"] == "stencil2d"
    p = np.pad(img, 2, mode="edge")
    total = np.zeros((n, m), np.float32)
    for i in range(5):
        acc = np.zeros((n, m), np.float32)
        for j in range(5):
            acc = (acc + (p[i:i + n, j:j + m] * w[i, j]).astype(np.float32)).astype(np.float32)
        total = (total + acc).astype(np.float32)
    np.testing.assert_array_equal(got.reshape(n, m), total)


@pytest.mark.parametrize("n,m", [(300, 516), (128, 128), (1000, 8), (4, 2052), (8192, 8192)])
def test_transpose_template_bit_exact(gpu, n, m):
    # the transpose2d template (TMA-swizzled 128 x 128 tiles); pitch % 4 == 0 sizes take it
    rng = np.random.default_rng(n + m)
    M = rng.standard_normal((n, m)).astype(np.float32)
    c = compile_program(PROGRAMS["transposeCopy"][0], None, name="transposeCopy")
    code = emit_cuda(c.unit)
    assert code.plan["stages"][0]["kind"] == "transpose2d"
    got = run_cuda(code, c.unit, {"n": n, "m": m}, [M], as_numpy=True)
    np.testing.assert_array_equal(got.reshape(m, n), M.T)


SLIDE5 = ("depFun((n: Nat) => fun(xs: Array[n, f32] => xs |> padClamp(2)(2) |> slide(5)(1) "
          "|> mapGlobal(fun(w => w |> reduceSeq(Private)(fun(a, v => a + v * 0.5f))(0.0f)))))")


@pytest.mark.parametrize("n", [4, 8, 4096, 4100, 8192 + 12, 1 << 20])
def test_stencil1d_template_bit_exact(gpu, n):
    # the stencil1d template (one bulk copy per 4096-output tile, padClamp in shared memory)
    rng = np.random.default_rng(n)
    xs = rng.standard_normal(n).astype(np.float32)
    c = compile_program(PROGRAMS["slide1D"][0], None, name="slide1D")
    code = emit_cuda(c.unit)
    assert code.plan["stages"][0]["kind"] == "stencil1d"
    got = run_cuda(code, c.unit, {"n": n}, [xs], as_numpy=True)
    p = np.pad(xs, (1, 1), mode="edge")
    want = ((np.float32(0) + p[:-2]) + p[1:-1]) + p[2:]
    np.testing.assert_array_equal(got, want.astype(np.float32))
    c5 = compile_program(SLIDE5, None, name="slide5")
    code5 = emit_cuda(c5.unit)
    assert code5.plan["stages"][0]["kind"] == "stencil1d"
    got5 = run_cuda(code5, c5.unit, {"n": n}, [xs], as_numpy=True)
    p5 = np.pad(xs, (2, 2), mode="edge")
    acc = np.zeros(n, np.float32)
    for k in range(5):
        acc = (acc + p5[k:k + n] * np.float32(0.5)).astype(np.float32)
    np.testing.assert_array_equal(got5, acc)


ROW3 = ("depFun((n: Nat, m: Nat) => fun(A: Array[n, Array[m, f32]] => fun(B: Array[n, Array[m, f32]] => "
        "fun(C: Array[n, Array[m, f32]] => zip(A)(zip(B)(C)) |> mapGlobal(fun(r => "
        "zip(fst(r))(zip(fst(snd(r)))(snd(snd(r)))) |> reduceSeq(Private)(fun(acc, t => "
        "acc + fst(t) * fst(snd(t)) * snd(snd(t))))(0.0f)))))))")


@pytest.mark.parametrize("n,m", [(8192, 512), (1000, 1028)])
def test_rowfold_three_row_streams_bit_exact(gpu, n, m):
    # three row streams: the ring depth shrinks to what fits two blocks per SM
    rng = np.random.default_rng(n)
    A, B, C = (rng.standard_normal((n, m)).astype(np.float32) for _ in range(3))
    c = compile_program(ROW3, None, name="row3")
    code = emit_cuda(c.unit)
    assert code.plan["stages"][0]["kind"] == "rowfold"
    got = run_cuda(code, c.unit, {"n": n, "m": m}, [A, B, C], as_numpy=True)
    acc = np.zeros(n, np.float32)
    for j in range(m):
        acc = (acc + (A[:, j] * B[:, j]) * C[:, j]).astype(np.float32)
    np.testing.assert_array_equal(got, acc)
