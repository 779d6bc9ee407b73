"""A vectorised restatement of the reference's functional semantics
(`interpreter.eval_program`, interpreter.py:81-260, plus the extension
primitives' denotations in paper_2201_03611_b200/extension.py §4) —
TEST INFRASTRUCTURE ONLY: the product path never imports it.

`eval_program` evaluates one value at a time in Python (≈ 15 µs per
element operation), which caps golden outputs at toy
sizes.  Here every `map` turns its array axis into a BATCH axis instead of
a Python loop: a value carries numpy arrays whose leading `nb` axes index
the independent instances being evaluated at once, and the closure body
runs once over all of them with numpy float32 arithmetic (IEEE binary32,
round to nearest — the same operations `eval_program` applies one by one).
`reduce` / `reduceSeq` stay left folds from `init` in element order (one
vectorised step per element), so results are BIT-IDENTICAL to
`eval_program` (pinned by tests/test_oracle.py on the reference's
END_TO_END programs and the configs' programs), but a 4096 x 4096 chunked
dot or a 1024² gemv evaluates in well under a second.

Representation (`Val`):
  kind "arr"  — numpy array `a`; axes [0, nb) are batch axes (possibly of
                size 1: broadcast), the rest are the value's own array axes
                (none for a scalar);
  kind "pair" — a tuple value (`a`, `b` are Vals);
  kind "zip"  — an array of tuples, stored as the two component arrays
                (struct of arrays; `a`, `b` are array Vals of equal length).
"""

from __future__ import annotations

import numpy as np

from paper_2201_03611_b200._ref import interpreter, nat, types
from paper_2201_03611_b200._ref import expr as _expr

Apply, DepApply, DepLambda, Identifier = _expr.Apply, _expr.DepApply, _expr.DepLambda, _expr.Identifier
Lambda, Literal, Primitive = _expr.Lambda, _expr.Literal, _expr.Primitive

ArrayType, ScalarType, TupleType = types.ArrayType, types.ScalarType, types.TupleType


class Val:
    __slots__ = ("kind", "a", "b", "nb")

    def __init__(self, kind, a, b=None, nb=0):
        self.kind, self.a, self.b, self.nb = kind, a, b, nb


def arr(a, nb):
    return Val("arr", a, None, nb)


# -- batch-depth bookkeeping -------------------------------------------------


def lift(v: Val, d: int) -> Val:
    """The same value seen from batch depth d >= v.nb (new singleton batch
    axes inserted after the existing ones)."""
    if v.nb == d:
        return v
    if v.kind == "arr":
        return arr(np.expand_dims(v.a, tuple(range(v.nb, d))), d)
    return Val(v.kind, lift(v.a, d), lift(v.b, d), d)


def length(v: Val) -> int:
    return v.a.shape[v.nb] if v.kind == "arr" else length(v.a)


def as_batch(v: Val) -> Val:
    """An array's elements as one batched value (the array axis becomes
    batch axis nb)."""
    if v.kind == "arr":
        return arr(v.a, v.nb + 1)
    return Val("pair", as_batch(v.a), as_batch(v.b), v.nb + 1)


def from_batch(v: Val, d: int, n: int) -> Val:
    """The inverse of as_batch: a value at depth d + 1 whose axis d has n
    entries becomes an array of n elements at depth d."""
    v = lift(v, d + 1)
    if v.kind == "arr":
        shape = list(v.a.shape)
        shape[d] = n
        return arr(np.broadcast_to(v.a, tuple(shape)), d)
    if v.kind == "pair":
        return Val("zip", from_batch(v.a, d, n), from_batch(v.b, d, n), d)
    return Val("zip", from_batch(v.a, d, n), from_batch(v.b, d, n), d)  # an array of arrays of tuples


def take(v: Val, i: int) -> Val:
    if v.kind == "arr":
        return arr(np.take(v.a, i, axis=v.nb), v.nb)
    return Val("pair", take(v.a, i), take(v.b, i), v.nb)


def on_axes(v: Val, fn) -> Val:
    """Apply an array-axis transformation (fn(numpy array, nb)) to every
    component of an array value."""
    if v.kind == "arr":
        return arr(fn(v.a, v.nb), v.nb)
    return Val("zip", on_axes(v.a, fn), on_axes(v.b, fn), v.nb)


# -- primitives ----------------------------------------------------------------


def _split(a, nb, s):
    n = a.shape[nb]
    if s <= 0 or n % s:
        raise interpreter.InterpreterError(f"cannot split array of length {n} by {s}")
    return a.reshape(a.shape[:nb] + (n // s, s) + a.shape[nb + 1:])


def _join(a, nb):
    return a.reshape(a.shape[:nb] + (a.shape[nb] * a.shape[nb + 1],) + a.shape[nb + 2:])


def _transpose(a, nb):
    return np.swapaxes(a, nb, nb + 1)


def _slide_idx(n, sz, sp):
    count = (n - sz) // sp + 1
    return np.arange(count)[:, None] * sp + np.arange(sz)[None, :]


def _slide(a, nb, sz, sp):  # extension.slide_values
    return np.take(a, _slide_idx(a.shape[nb], sz, sp), axis=nb)


def _pad_clamp(a, nb, lo, hi):  # extension.pad_clamp_values
    n = a.shape[nb]
    return np.take(a, np.clip(np.arange(lo + n + hi) - lo, 0, n - 1), axis=nb)


def _slide2d(a, nb, sz, sp):  # extension.slide2d_values: [rows][cols] -> [rw][cw][sz][sz]
    a = _slide(a, nb + 1, sz, sp)  # [n_r][cw][sz_c]
    a = _slide(a, nb, sz, sp)  # [rw][sz_r][cw][sz_c]
    return np.swapaxes(a, nb + 1, nb + 2)


def _binop(name, x: Val, y: Val) -> Val:
    d = max(x.nb, y.nb)
    a, b = lift(x, d).a, lift(y, d).a
    if a.dtype == np.float32 or b.dtype == np.float32:  # interpreter.py:161-169
        a, b = a.astype(np.float32, copy=False), b.astype(np.float32, copy=False)
        with np.errstate(all="ignore"):
            if name == "add":
                return arr(a + b, d)
            if name == "sub":
                return arr(a - b, d)
            if name == "mul":
                return arr(a * b, d)
            if name == "div":
                return arr(a / b, d)
    if name == "add":
        return arr(a + b, d)
    if name == "sub":
        return arr(a - b, d)
    if name == "mul":
        return arr(a * b, d)
    if name == "div":  # extension.f32_div on integers: truncation toward zero
        q = np.abs(a) // np.abs(b)
        return arr(np.where((a >= 0) == (b >= 0), q, -q), d)
    raise AssertionError(name)


_ARITY = dict(interpreter._PRIM_ARITY)
_ARITY.update({"transpose": 1, "slide": 1, "padClamp": 1, "padClamp2D": 1, "slide2D": 1,
               "div": 2, "sqrt": 1, "rsqrt": 1, "abs": 1, "toGlobal": 1, "toLocal": 1, "toPrivate": 1})
_IDENTITY = {"toMem", "id", "toGlobal", "toLocal", "toPrivate"}


class Closure:
    def __init__(self, param, body, env):
        self.param, self.body, self.env = param, body, env


class DepClosure:
    def __init__(self, param, body, env, nat_env):
        self.param, self.body, self.env, self.nat_env = param, body, env, nat_env


class Partial:
    def __init__(self, name, deps, args):
        self.name, self.deps, self.args = name, deps, args


def eval_expr(e, env, nat_env, depth=0):
    """`depth`: the number of batch axes of the evaluation context (the
    enclosing maps); a `map` met here adds batch axis `depth`."""
    if isinstance(e, Identifier):
        return env[e.uid]
    if isinstance(e, Literal):
        if isinstance(e.value, bool):
            return arr(np.asarray(e.value), 0)
        if isinstance(e.value, float):
            return arr(np.asarray(np.float32(e.value)), 0)
        return arr(np.asarray(e.value, dtype=np.int64), 0)
    if isinstance(e, Lambda):
        return Closure(e.param, e.body, env)
    if isinstance(e, DepLambda):
        return DepClosure(e.param, e.body, env, nat_env)
    if isinstance(e, Primitive):
        return Partial(e.name, [], [])
    if isinstance(e, Apply):
        return apply_value(eval_expr(e.fn, env, nat_env, depth), eval_expr(e.arg, env, nat_env, depth), nat_env, depth)
    if isinstance(e, DepApply):
        arg = e.arg
        if isinstance(arg, nat.Nat):
            arg = nat.evaluate(arg, nat_env)
        return apply_dep(eval_expr(e.fn, env, nat_env, depth), arg, nat_env, depth)
    raise interpreter.InterpreterError(f"cannot evaluate {e!r}")


def apply_value(f, a, nat_env, depth):
    if isinstance(f, Closure):
        return eval_expr(f.body, {**f.env, f.param.uid: a}, nat_env, depth)
    if isinstance(f, Partial):
        args = f.args + [a]
        if len(args) == _ARITY[f.name]:
            return exec_prim(f.name, f.deps, args, nat_env, depth)
        return Partial(f.name, f.deps, args)
    raise interpreter.InterpreterError(f"cannot apply {f!r}")


def apply_dep(f, x, nat_env, depth):
    if isinstance(f, DepClosure):
        return eval_expr(f.body, f.env, {**f.nat_env, f.param: x}, depth)
    if isinstance(f, Partial):
        return Partial(f.name, f.deps + [x], f.args)
    raise interpreter.InterpreterError(f"cannot apply {f!r}")


def exec_prim(name, deps, args, nat_env, depth):
    if name in ("map", "mapSeq", "mapGlobal", "mapWorkGroup", "mapLocal"):
        f, xs = args
        xs = lift(xs, depth)  # its array axis becomes batch axis `depth`
        return from_batch(apply_value(f, as_batch(xs), nat_env, depth + 1), depth, length(xs))
    if name in ("reduce", "reduceSeq", "reduceSeqIn"):  # a left fold from init, in element order
        op, acc, xs = args
        xs = lift(xs, depth)
        for i in range(length(xs)):
            acc = apply_value(apply_value(op, acc, nat_env, depth), take(xs, i), nat_env, depth)
        return acc
    if name == "zip":
        a, b = args
        d = max(a.nb, b.nb)
        a, b = lift(a, d), lift(b, d)
        if length(a) != length(b):
            raise interpreter.InterpreterError("zip of arrays with different lengths")
        return Val("zip", a, b, d)
    if name in ("fst", "snd"):
        (p,) = args
        return p.a if name == "fst" else p.b
    if name in ("split", "asVector"):  # asVector(w) is split(w) as a value (extension.py)
        return on_axes(args[0], lambda a, nb: _split(a, nb, deps[0]))
    if name in ("join", "asScalar"):
        return on_axes(args[0], _join)
    if name == "transpose":
        return on_axes(args[0], _transpose)
    if name == "slide":
        return on_axes(args[0], lambda a, nb: _slide(a, nb, *deps))
    if name == "padClamp":
        return on_axes(args[0], lambda a, nb: _pad_clamp(a, nb, *deps))
    if name == "padClamp2D":
        return on_axes(args[0], lambda a, nb: _pad_clamp(_pad_clamp(a, nb + 1, *deps), nb, *deps))
    if name == "slide2D":
        return on_axes(args[0], lambda a, nb: _slide2d(a, nb, *deps))
    if name in _IDENTITY:
        return args[0]
    if name in ("add", "sub", "mul", "div"):
        return _binop(name, *args)
    if name in ("sqrt", "rsqrt", "abs"):
        (x,) = args
        with np.errstate(all="ignore"):
            if name == "abs":
                return arr(np.abs(x.a), x.nb)
            s = np.sqrt(x.a.astype(np.float32, copy=False))
            return arr(s if name == "sqrt" else np.float32(1.0) / s, x.nb)
    if name == "iterate":  # interpreter.py:170-184
        (k,) = deps
        f, xs = args
        step = interpreter._iterate_shrink_factor(_as_ref_depclosure(f), nat_env)
        current = xs
        for _ in range(k):
            l_val = length(current) // step
            current = apply_value(apply_dep(f, l_val, nat_env, depth), current, nat_env, depth)
        return current
    raise interpreter.InterpreterError(f"no vectorised denotation for primitive {name!r}")


def _as_ref_depclosure(f):
    return interpreter.DepClosure(f.param, f.body, f.env, f.nat_env)


# -- programs ------------------------------------------------------------------


def convert_input(raw, dtype) -> Val:
    if isinstance(dtype, ArrayType) and isinstance(_innermost(dtype), TupleType):
        if isinstance(dtype.elem, TupleType):
            fst = [r[0] for r in raw]
            snd = [r[1] for r in raw]
            return Val("zip", convert_input(fst, ArrayType(dtype.size, dtype.elem.fst)),
                       convert_input(snd, ArrayType(dtype.size, dtype.elem.snd)), 0)
        raise interpreter.InterpreterError("nested arrays of tuples are not supported here")
    if isinstance(dtype, TupleType):
        return Val("pair", convert_input(raw[0], dtype.fst), convert_input(raw[1], dtype.snd), 0)
    scalar = _innermost(dtype)
    np_t = np.float32 if scalar == types.F32 else (np.bool_ if scalar == types.BOOL else np.int64)
    return arr(np.asarray(raw, dtype=np_t), 0)


def _innermost(t):
    while isinstance(t, ArrayType):
        t = t.elem
    return t


def eval_program(e, nat_assignment: dict, inputs) -> Val:
    """Same contract as interpreter.eval_program (interpreter.py:223-245);
    inputs may be nested lists or numpy arrays."""
    nat_env = dict(nat_assignment)
    env = {}
    inputs = list(inputs)
    while True:
        if isinstance(e, DepLambda):
            e = e.body
        elif isinstance(e, Lambda):
            env[e.param.uid] = convert_input(inputs.pop(0), e.param.type)
            e = e.body
        else:
            break
    return eval_expr(e, env, nat_env)


def to_numpy(v: Val):
    """A depth-0 value as numpy (arrays of tuples: a pair of arrays)."""
    if v.kind == "arr":
        return np.ascontiguousarray(v.a)
    return (to_numpy(v.a), to_numpy(v.b))


def to_plain(v: Val):
    """A depth-0 value as the nested lists / floats interpreter.to_plain gives."""
    if v.kind == "arr":
        return v.a.tolist()
    if v.kind == "pair":
        return [to_plain(v.a), to_plain(v.b)]
    left, right = to_plain(v.a), to_plain(v.b)
    return [[x, y] for x, y in zip(left, right)]
