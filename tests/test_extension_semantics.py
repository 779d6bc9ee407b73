"""the primitives the reference lacks (transpose, slide,
slide2D, padClamp, padClamp2D, asVector / asScalar, abs, div, sqrt, rsqrt)
have no reference oracle, so their denotations (extension.py) are pinned
here against independent standard definitions: numpy's `transpose`,
`pad(mode="edge")` (clamp-to-edge padding), `sliding_window_view` and
IEEE binary32 arithmetic — evaluated through the reference's OWN
interpreter (`eval_program`, with the extension registered through its
seams) on random inputs and sizes."""

import random

import numpy as np
import pytest
from numpy.lib.stride_tricks import sliding_window_view

from paper_2201_03611_b200._ref import interpreter, nat
from paper_2201_03611_b200.frontend import typed_program


def _eval(src, nats, inputs, assumptions=()):
    _name, typed, _free = typed_program(src, assumptions)
    return np.asarray(interpreter.to_plain(interpreter.eval_program(typed, nats, inputs)), np.float32)


def _mat(rng, n, m):
    return np.asarray([[np.float32(rng.uniform(-4, 4)) for _ in range(m)] for _ in range(n)], np.float32)


@pytest.mark.parametrize("n,m", [(1, 1), (3, 5), (7, 2)])
def test_transpose_is_numpy_transpose(n, m):
    M = _mat(random.Random(n * 10 + m), n, m)
    src = ("depFun((n: Nat, m: Nat) => fun(M: Array[n, Array[m, f32]] => "
           "M |> transpose |> map(map(fun(v => v * 1.0f)))))")
    np.testing.assert_array_equal(_eval(src, {"n": n, "m": m}, [M.tolist()]), M.T)


@pytest.mark.parametrize("n,l,r", [(1, 1, 1), (5, 2, 0), (6, 0, 3), (4, 3, 3)])
def test_pad_clamp_is_edge_padding(n, l, r):
    xs = _mat(random.Random(n + l * 7 + r), 1, n)[0]
    src = f"depFun((n: Nat) => fun(xs: Array[n, f32] => xs |> padClamp({l})({r}) |> map(fun(v => v * 1.0f))))"
    np.testing.assert_array_equal(_eval(src, {"n": n}, [xs.tolist()]), np.pad(xs, (l, r), mode="edge"))


@pytest.mark.parametrize("n,m,l,r", [(1, 1, 1, 1), (3, 4, 1, 2), (5, 2, 2, 0)])
def test_pad_clamp_2d_is_edge_padding(n, m, l, r):
    M = _mat(random.Random(n * m + l), n, m)
    src = (f"depFun((n: Nat, m: Nat) => fun(M: Array[n, Array[m, f32]] => "
           f"M |> padClamp2D({l})({r}) |> map(map(fun(v => v * 1.0f)))))")
    np.testing.assert_array_equal(_eval(src, {"n": n, "m": m}, [M.tolist()]), np.pad(M, ((l, r), (l, r)), mode="edge"))


@pytest.mark.parametrize("sz,sp,count", [(3, 1, 5), (2, 2, 4), (4, 3, 3), (1, 1, 6)])
def test_slide_is_a_strided_sliding_window(sz, sp, count):
    length = sp * (count - 1) + sz
    xs = _mat(random.Random(sz * 31 + sp), 1, length)[0]
    src = (f"depFun((n: Nat) => fun(xs: Array[{sp} * n + {sz}, f32] => "
           f"xs |> slide({sz})({sp}) |> map(map(fun(v => v * 1.0f)))))")
    got = _eval(src, {"n": count - 1}, [xs.tolist()])
    np.testing.assert_array_equal(got, sliding_window_view(xs, sz)[::sp])


@pytest.mark.parametrize("sz,sp,rows,cols", [(3, 1, 4, 5), (2, 2, 3, 2), (3, 2, 2, 3)])
def test_slide_2d_windows_are_numpy_windows(sz, sp, rows, cols):
    n, m = sp * (rows - 1) + sz, sp * (cols - 1) + sz
    M = _mat(random.Random(n * 100 + m), n, m)
    src = (f"depFun((a: Nat, b: Nat) => fun(M: Array[{sp} * a + {sz}, Array[{sp} * b + {sz}, f32]] => "
           f"M |> slide2D({sz})({sp}) |> map(map(map(map(fun(v => v * 1.0f)))))))")
    got = _eval(src, {"a": rows - 1, "b": cols - 1}, [M.tolist()])
    want = sliding_window_view(M, (sz, sz))[::sp, ::sp]  # [i, j, a, b] = M[i*sp + a, j*sp + b]
    np.testing.assert_array_equal(got, want)


def test_vector_views_are_split_and_join():
    xs = _mat(random.Random(3), 1, 12)[0]
    src = "depFun((n: Nat) => fun(xs: Array[n, f32] => xs |> asVector(4) |> map(map(fun(v => v * 1.0f)))))"
    got = _eval(src, {"n": 12}, [xs.tolist()], assumptions=[(nat.Var("n"), nat.Const(4))])
    np.testing.assert_array_equal(got, xs.reshape(3, 4))
    src = ("depFun((n: Nat, m: Nat) => fun(M: Array[n, Array[m, f32]] => "
           "M |> asScalar |> map(fun(v => v * 1.0f))))")
    M = xs.reshape(3, 4)
    np.testing.assert_array_equal(_eval(src, {"n": 3, "m": 4}, [M.tolist()]), xs)


def test_scalar_functions_are_ieee_binary32():
    rng = random.Random(5)
    a = np.asarray([np.float32(rng.uniform(0.01, 9)) for _ in range(64)], np.float32)
    b = np.asarray([np.float32(rng.uniform(-9, 9)) for _ in range(64)], np.float32)
    src = ("depFun((n: Nat) => fun(a: Array[n, f32] => fun(b: Array[n, f32] => zip(a)(b) |> map(fun(p => "
           "div(abs(snd(p)))(fst(p)) + sqrt(fst(p)) * rsqrt(fst(p)))))))")
    got = _eval(src, {"n": 64}, [a.tolist(), b.tolist()])
    with np.errstate(all="ignore"):
        q = (np.abs(b) / a).astype(np.float32)
        sq = np.sqrt(a).astype(np.float32)
        rs = (np.float32(1) / np.sqrt(a).astype(np.float32)).astype(np.float32)
        want = (q + (sq * rs).astype(np.float32)).astype(np.float32)
    np.testing.assert_array_equal(got, want)
