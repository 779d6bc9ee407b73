"""New primitives for the north-star patterns, registered through the
reference's own extension seams (SURVEY.md §8 b, last row; §8.1).

The reference lacks `transpose`, `slide`, `slide2D`, `padClamp`,
`padClamp2D`, `div`, `sqrt`, `rsqrt` and Shine's `toGlobal/toLocal/toPrivate`
spellings.  Each is added in four places, and nowhere else:

1. typing    — `Registry.register_scheme`            (primitives.py:76)
2. DPIA      — `dpia.SIGNATURES` / `SIGNATURE_TEXT`  (dpia.py:230-349)
3. lowering  — `lowering._targs_for` (wrapped; it is an if-chain,
               lowering.py:222-255) and `_ACC_CASES` / `_CON_CASES`
               (lowering.py:557-585)
4. oracle    — `interpreter._PRIM_ARITY` + `_exec_prim` (interpreter.py:58-185)
               for `eval_program`, and `_eval_fun_prim` / `eval_acc_phrase`
               (interpreter.py:491-564) for `run_unit`.
5. C emitter — `codegen.emit_exp` / `emit_acc` (codegen.py:179-290, module
               functions that recurse through their globals, so a wrapper
               sees every level) and `codegen.emit` (helpers), so the
               reference's own C / OpenMP emission covers the programs that
               use them (the CPU baseline and full-size oracle of conv and
               nbody, oracle/make_ref.py).
6. rules     — `rules.RULES` / `RULE_PARAMS` (rules.py:237-259): the
               GPU-oriented rewrite rules of gpu_rules.py for strategy files.

Semantics (there is no reference oracle for these — "parity unpinned" for
them in the sense of SURVEY.md §8 c; these definitions are the spec):

* `slide(sz)(sp)`: Array[sp*n+sz, t] -> Array[n+1, Array[sz, t]],
  window i = xs[i*sp : i*sp+sz].
* `padClamp(l)(r)`: Array[n, t] -> Array[l+n+r, t], index k reads
  xs[clamp(k-l, 0, n-1)].
* `padClamp2D(l)(r)` = map(padClamp(l)(r)) >> padClamp(l)(r).
* `slide2D(sz)(sp)` = map(slide(sz)(sp)) >> slide(sz)(sp) >> map(transpose):
  window (i, j) row a col b = xs[i*sp+a][j*sp+b].
* `transpose`: Array[n, Array[m, t]] -> Array[m, Array[n, t]].
* `abs` is |x| (exact: the sign bit cleared for binary32; i32 abs).
* `div` is IEEE binary32 division (C truncation for i32); `sqrt` is IEEE
  binary32 square root; `rsqrt(x)` = 1.0f / sqrt(x) with both operations
  rounded to binary32 (the GPU evaluates it with the MUFU reciprocal square
  root, so programs using it are compared under a tolerance).
* `toGlobal/toLocal/toPrivate` = `toMem(Global/Local/Private)`.
* `asVector(w)`: Array[w*q, t] -> Array[q, Array[w, t]] and `asScalar`:
  Array[a, Array[b, t]] -> Array[a*b, t] — Shine's vector views
  (PAPER.md:1047-1051): as values they are split(w) / join; as memory
  accesses they promise that the w elements of a vector are contiguous
  and w-aligned, so the sm100a emitter reads / writes them as one float2 /
  float4 (emit_cuda.GenericKernel, `vectorize`).
"""

from __future__ import annotations

import dataclasses
import re

import numpy as np

from ._ref import codegen, dpia, errors, interpreter, lowering, nat, primitives, rules
from .types_util import array_elem

# ---------------------------------------------------------------------------
# 1. typing

SCHEMES = {
    "transpose": "{n: Nat} -> {m: Nat} -> {t: DataType} -> Array[n, Array[m, t]] -> Array[m, Array[n, t]]",
    "slide": "(sz: Nat) -> (sp: Nat) -> {n: Nat} -> {t: DataType} -> Array[sp * n + sz, t] -> Array[n + 1, Array[sz, t]]",
    "padClamp": "(l: Nat) -> (r: Nat) -> {n: Nat} -> {t: DataType} -> Array[n, t] -> Array[l + n + r, t]",
    "padClamp2D": "(l: Nat) -> (r: Nat) -> {n: Nat} -> {m: Nat} -> {t: DataType} -> Array[n, Array[m, t]] -> Array[l + n + r, Array[l + m + r, t]]",
    "slide2D": "(sz: Nat) -> (sp: Nat) -> {n: Nat} -> {m: Nat} -> {t: DataType} -> Array[sp * n + sz, Array[sp * m + sz, t]] -> Array[n + 1, Array[m + 1, Array[sz, Array[sz, t]]]]",
    "div": "{t: DataType} -> t -> t -> t",
    "sqrt": "{t: DataType} -> t -> t",
    "rsqrt": "{t: DataType} -> t -> t",
    "abs": "{t: DataType} -> t -> t",
    "toGlobal": "{t: DataType} -> t -> t",
    "toLocal": "{t: DataType} -> t -> t",
    "toPrivate": "{t: DataType} -> t -> t",
    "asVector": "(w: Nat) -> {q: Nat} -> {t: DataType} -> Array[w * q, t] -> Array[q, Array[w, t]]",
    "asScalar": "{a: Nat} -> {b: Nat} -> {t: DataType} -> Array[a, Array[b, t]] -> Array[a * b, t]",
}

# ---------------------------------------------------------------------------
# 2. DPIA signatures (same notation as dpia.SIGNATURE_TEXT)

SIGNATURE_TEXT = {
    "transpose": "(n: Nat, m: Nat, t: DataType, w: ReadWrite, x: Exp[Array[n,Array[m,t]],w]): Exp[Array[m,Array[n,t]],w]",
    "slide": "(sz: Nat, sp: Nat, n: Nat, t: DataType, x: Exp[Array[sp*n+sz,t],Rd]): Exp[Array[n+1,Array[sz,t]],Rd]",
    "padClamp": "(l: Nat, r: Nat, n: Nat, t: DataType, x: Exp[Array[n,t],Rd]): Exp[Array[l+n+r,t],Rd]",
    "padClamp2D": "(l: Nat, r: Nat, n: Nat, m: Nat, t: DataType, x: Exp[Array[n,Array[m,t]],Rd]): Exp[Array[l+n+r,Array[l+m+r,t]],Rd]",
    "slide2D": "(sz: Nat, sp: Nat, n: Nat, m: Nat, t: DataType, x: Exp[Array[sp*n+sz,Array[sp*m+sz,t]],Rd]): Exp[Array[n+1,Array[m+1,Array[sz,Array[sz,t]]]],Rd]",
    "div": "(t: DataType, w: ReadWrite, a: Exp[t,Rd], b: Exp[t,Rd]): Exp[t,w]",
    "sqrt": "(t: DataType, w: ReadWrite, a: Exp[t,Rd]): Exp[t,w]",
    "rsqrt": "(t: DataType, w: ReadWrite, a: Exp[t,Rd]): Exp[t,w]",
    "abs": "(t: DataType, w: ReadWrite, a: Exp[t,Rd]): Exp[t,w]",
    "toGlobal": "(t: DataType, x: Exp[t,Wr]): Exp[t,Rd]",
    "toLocal": "(t: DataType, x: Exp[t,Wr]): Exp[t,Rd]",
    "toPrivate": "(t: DataType, x: Exp[t,Wr]): Exp[t,Rd]",
    # imperative: the acceptor view written through by accT(transpose)
    "transposeAcc": "(n: Nat, m: Nat, t: DataType, array: Acc[Array[m,Array[n,t]]]): Acc[Array[n,Array[m,t]]]",
    # vector views: split / join with the same index maps (dpia.py:240-241, 259-260)
    "asVector": "(n: Nat, m: Nat, t: DataType, w: ReadWrite, x: Exp[Array[n*m,t],w]): Exp[Array[m,Array[n,t]],w]",
    "asScalar": "(n: Nat, m: Nat, t: DataType, w: ReadWrite, x: Exp[Array[n,Array[m,t]],w]): Exp[Array[n*m,t],w]",
    "asVectorAcc": "(n: Nat, m: Nat, t: DataType, array: Acc[Array[m,Array[n,t]]]): Acc[Array[n*m,t]]",
    "asScalarAcc": "(n: Nat, m: Nat, t: DataType, array: Acc[Array[n*m,t]]): Acc[Array[n,Array[m,t]]]",
}
# each vector view and acceptor behaves as its split / join counterpart
VECTOR_AS = {"asVector": "split", "asScalar": "join", "asVectorAcc": "splitAcc", "asScalarAcc": "joinAcc"}

VIEW_TAGS = ("transpose", "slide", "padClamp", "padClamp2D", "slide2D")
BINARY_TAGS = ("div",)
UNARY_TAGS = ("sqrt", "rsqrt", "abs")
TO_MEM_ALIASES = {"toGlobal": "Global", "toLocal": "Local", "toPrivate": "Private"}

_installed = False


def install(registry=None):
    """Register every extension primitive (idempotent)."""
    global _installed
    registry = registry or primitives.default_registry()
    for name, scheme in SCHEMES.items():
        if name not in registry:
            registry.register_scheme(name, scheme)
    if _installed:
        return registry
    for tag, text in SIGNATURE_TEXT.items():
        dpia.SIGNATURE_TEXT[tag] = text
        dpia.SIGNATURES[tag] = dpia._parse_signature(tag, text)
    _install_lowering()
    _install_interpreter()
    _install_c_emitter()
    from . import gpu_rules

    gpu_rules.install(rules)  # 6. GPU-oriented rewrite rules (gpu_rules.py)
    _installed = True
    return registry


# ---------------------------------------------------------------------------
# 3. lowering


def _install_lowering():
    AddressSpace = lowering.AddressSpace

    base_targs = lowering._targs_for

    def targs_for(tag, vt, deps, ctx):
        slots, out = lowering._fun_slots(vt)
        if tag == "transpose":
            arr = slots[0]
            return (arr.size, arr.elem.size, arr.elem.elem, dpia.RWVar(lowering._fresh_rw(ctx)))
        if tag == "slide":
            sz, sp = deps
            n = nat.normalize(out.size - nat.Const(1))
            return (sz, sp, n, out.elem.elem)
        if tag == "padClamp":
            l, r = deps
            return (l, r, slots[0].size, slots[0].elem)
        if tag == "padClamp2D":
            l, r = deps
            arr = slots[0]
            return (l, r, arr.size, arr.elem.size, arr.elem.elem)
        if tag == "slide2D":
            sz, sp = deps
            n = nat.normalize(out.size - nat.Const(1))
            m = nat.normalize(out.elem.size - nat.Const(1))
            return (sz, sp, n, m, array_elem(out, 4))
        if tag in BINARY_TAGS or tag in UNARY_TAGS:
            return (out, dpia.RWVar(lowering._fresh_rw(ctx)))
        if tag in TO_MEM_ALIASES:
            return (out,)
        if tag in ("asVector", "asScalar"):
            return base_targs(VECTOR_AS[tag], vt, deps, ctx)
        return base_targs(tag, vt, deps, ctx)

    lowering._targs_for = targs_for

    def acc_transpose(ctx, expr, output):
        n, m, t, _w = expr.type_args
        (arr,) = expr.args
        view = dpia.ImpPrim(
            "transposeAcc", (n, m, t), (output,),
            dpia.AccType(lowering.ArrayType(n, lowering.ArrayType(m, t))),
        )
        return lowering.acc_t(ctx, arr, view)

    def acc_unop(ctx, expr, output):
        t, _w = expr.type_args

        def done(a):
            return lowering._assign(t, output, dpia.FunPrim(expr.tag, (t, dpia.RD), (a,), dpia.ExpType(t, dpia.RD)))

        return lowering.con_t(ctx, expr.args[0], done)

    def con_unop(ctx, expr, k):
        t, _w = expr.type_args
        return lowering.con_t(
            ctx, expr.args[0],
            lambda a: k(dpia.FunPrim(expr.tag, (t, dpia.RD), (a,), dpia.ExpType(t, dpia.RD))),
        )

    def con_to_mem_alias(space):
        def handler(ctx, expr, k):
            (t,) = expr.type_args
            (value,) = expr.args

            def body(tmp_e, tmp_a):
                return lowering._seq(lowering.acc_t(ctx, value, tmp_a), k(tmp_e))

            return lowering._new(ctx, space, t, "tmp", body)

        return handler

    def acc_vector(acc_tag):
        # accT(asVector(x)) / accT(asScalar(x)): x written through the dual
        # acceptor (lowering.py:404-417 with the vector tags)
        def handler(ctx, expr, output):
            n, m, t, _w = expr.type_args
            (arr,) = expr.args
            shape = (lowering.ArrayType(nat.normalize(n * m), t) if acc_tag == "asVectorAcc"
                     else lowering.ArrayType(n, lowering.ArrayType(m, t)))
            view = dpia.ImpPrim(acc_tag, (n, m, t), (output,), dpia.AccType(shape))
            return lowering.acc_t(ctx, arr, view)

        return handler

    for tag in VIEW_TAGS + ("asVector", "asScalar"):
        lowering._CON_CASES[tag] = lowering._con_passthrough
    lowering._ACC_CASES["asVector"] = acc_vector("asVectorAcc")
    lowering._ACC_CASES["asScalar"] = acc_vector("asScalarAcc")
    lowering._ACC_CASES["transpose"] = acc_transpose
    for tag in BINARY_TAGS:
        lowering._ACC_CASES[tag] = lowering._acc_binop
        lowering._CON_CASES[tag] = lowering._con_binop
    for tag in UNARY_TAGS:
        lowering._ACC_CASES[tag] = acc_unop
        lowering._CON_CASES[tag] = con_unop
    for tag, space in TO_MEM_ALIASES.items():
        lowering._CON_CASES[tag] = con_to_mem_alias(AddressSpace(space))


# ---------------------------------------------------------------------------
# 4. oracle semantics


def _clamp(k, n):
    return 0 if k < 0 else (n - 1 if k > n - 1 else k)


def slide_values(xs, sz, sp):
    count = (len(xs) - sz) // sp + 1
    return [list(xs[i * sp: i * sp + sz]) for i in range(count)]


def pad_clamp_values(xs, l, r):
    n = len(xs)
    return [xs[_clamp(k - l, n)] for k in range(l + n + r)]


def transpose_values(xs):
    if not xs:
        return []
    return [list(col) for col in zip(*xs)]


def pad_clamp2d_values(xs, l, r):
    return pad_clamp_values([pad_clamp_values(row, l, r) for row in xs], l, r)


def slide2d_values(xs, sz, sp):
    rows = slide_values([slide_values(row, sz, sp) for row in xs], sz, sp)
    return [transpose_values(band) for band in rows]


def f32_div(a, b):
    if isinstance(a, np.float32) or isinstance(b, np.float32):
        with np.errstate(all="ignore"):
            return np.float32(a) / np.float32(b)
    q = abs(a) // abs(b)
    return q if (a >= 0) == (b >= 0) else -q


def f32_sqrt(a):
    with np.errstate(all="ignore"):
        return np.sqrt(np.float32(a))


def f32_rsqrt(a):
    with np.errstate(all="ignore"):
        return np.float32(1.0) / np.sqrt(np.float32(a))


def any_abs(a):
    """|a|: exact for binary32 (sign bit cleared) and i32."""
    if isinstance(a, np.float32):
        return np.float32(abs(a))
    return abs(a)


def _install_interpreter():
    arity = {"transpose": 1, "slide": 1, "padClamp": 1, "padClamp2D": 1, "slide2D": 1,
             "div": 2, "sqrt": 1, "rsqrt": 1, "abs": 1, "toGlobal": 1, "toLocal": 1, "toPrivate": 1,
             "asVector": 1, "asScalar": 1}
    interpreter._PRIM_ARITY.update(arity)
    base_exec = interpreter._exec_prim

    def exec_prim(name, deps, args, nat_env):
        if name == "transpose":
            return transpose_values(args[0])
        if name == "slide":
            sz, sp = deps
            return slide_values(args[0], sz, sp)
        if name == "padClamp":
            l, r = deps
            return pad_clamp_values(args[0], l, r)
        if name == "padClamp2D":
            l, r = deps
            return pad_clamp2d_values(args[0], l, r)
        if name == "slide2D":
            sz, sp = deps
            return slide2d_values(args[0], sz, sp)
        if name == "div":
            return f32_div(*args)
        if name == "sqrt":
            return f32_sqrt(args[0])
        if name == "rsqrt":
            return f32_rsqrt(args[0])
        if name == "abs":
            return any_abs(args[0])
        if name in TO_MEM_ALIASES:
            return args[0]
        if name in ("asVector", "asScalar"):
            return base_exec(VECTOR_AS[name], deps, args, nat_env)
        return base_exec(name, deps, args, nat_env)

    interpreter._exec_prim = exec_prim

    base_fun = interpreter._eval_fun_prim

    def eval_fun_prim(p, env, store, nat_env):
        tag = p.tag
        ev = interpreter.eval_exp_phrase
        if tag in VIEW_TAGS:
            xs = ev(p.args[0], env, store, nat_env)
            if tag == "transpose":
                return transpose_values(xs)
            a = nat.evaluate(p.type_args[0], nat_env)
            b = nat.evaluate(p.type_args[1], nat_env)
            return {"slide": slide_values, "padClamp": pad_clamp_values,
                    "padClamp2D": pad_clamp2d_values, "slide2D": slide2d_values}[tag](xs, a, b)
        if tag == "div":
            return f32_div(ev(p.args[0], env, store, nat_env), ev(p.args[1], env, store, nat_env))
        if tag == "sqrt":
            return f32_sqrt(ev(p.args[0], env, store, nat_env))
        if tag == "rsqrt":
            return f32_rsqrt(ev(p.args[0], env, store, nat_env))
        if tag == "abs":
            return any_abs(ev(p.args[0], env, store, nat_env))
        if tag in ("asVector", "asScalar"):
            return base_fun(dataclasses.replace(p, tag=VECTOR_AS[tag]), env, store, nat_env)
        return base_fun(p, env, store, nat_env)

    interpreter._eval_fun_prim = eval_fun_prim

    base_acc = interpreter.eval_acc_phrase

    def eval_acc_phrase(p, env, store, nat_env):
        if isinstance(p, dpia.ImpPrim) and p.tag == "transposeAcc":
            base = eval_acc_phrase(p.args[0], env, store, nat_env).resolve(store)
            return base.via(lambda tail: (tail[1], tail[0]) + tail[2:])
        if isinstance(p, dpia.ImpPrim) and p.tag in ("asVectorAcc", "asScalarAcc"):
            return base_acc(dataclasses.replace(p, tag=VECTOR_AS[p.tag]), env, store, nat_env)
        return base_acc(p, env, store, nat_env)

    interpreter.eval_acc_phrase = eval_acc_phrase


# ---------------------------------------------------------------------------
# 5. C emission (the reference's C / OpenMP targets)

C_HELPERS = """static inline int rs_clamp(int k, int hi) { return k < 0 ? 0 : (k > hi ? hi : k); }
"""


def _clamp_nat(k, hi, state):
    """A clamped index as a nat atom: nat.py has no min/max node (SURVEY.md
    §8.1), so the clamp is an opaque variable whose name IS its C text
    (codegen._render prints a Var's name verbatim); normalisation keeps it as
    an atom, and equal clamps share one atom."""
    inner = codegen._render_nat(k, state)
    return nat.Var(f"rs_clamp({inner}, {codegen._render_nat(nat.normalize(hi - nat.Const(1)), state)})")


def _install_c_emitter():
    base_exp = codegen.emit_exp
    base_acc = codegen.emit_acc
    base_emit = codegen.emit

    def emit_exp(p, env, state, pending=(), projs=()):
        if isinstance(p, dpia.FunPrim) and p.tag in VIEW_TAGS:
            x = p.args[0]
            ta = p.type_args
            if p.tag == "transpose":
                i, j, *rest = pending
                return emit_exp(x, env, state, (j, i, *rest), projs)
            if p.tag == "slide":
                sp = ta[1]
                i, a, *rest = pending
                return emit_exp(x, env, state, (i * sp + a, *rest), projs)
            if p.tag == "slide2D":
                sp = ta[1]
                i, j, a, b, *rest = pending
                return emit_exp(x, env, state, (i * sp + a, j * sp + b, *rest), projs)
            if p.tag == "padClamp":
                l, _r, n = ta[0], ta[1], ta[2]
                k, *rest = pending
                return emit_exp(x, env, state, (_clamp_nat(k - l, n, state), *rest), projs)
            if p.tag == "padClamp2D":
                l, _r, n, m = ta[0], ta[1], ta[2], ta[3]
                i, j, *rest = pending
                return emit_exp(x, env, state, (_clamp_nat(i - l, n, state), _clamp_nat(j - l, m, state), *rest),
                                projs)
        if isinstance(p, dpia.FunPrim) and p.tag in ("asVector", "asScalar"):
            return emit_exp(dataclasses.replace(p, tag=VECTOR_AS[p.tag]), env, state, pending, projs)
        if isinstance(p, dpia.FunPrim) and p.tag in BINARY_TAGS + UNARY_TAGS:
            if pending or projs:
                raise errors.EmitError("indexed arithmetic value")
            a = emit_exp(p.args[0], env, state)
            if p.tag == "div":
                return f"({a} / {emit_exp(p.args[1], env, state)})"
            if p.tag == "sqrt":
                return f"sqrtf({a})"
            if p.tag == "abs":
                t = p.type_args[0]
                return f"fabsf({a})" if getattr(t, "name", "f32") == "f32" else f"abs({a})"
            return f"(1.0f / sqrtf({a}))"  # rsqrt: both operations rounded to binary32
        return base_exp(p, env, state, pending, projs)

    def emit_acc(p, env, state, pending=()):
        if isinstance(p, dpia.ImpPrim) and p.tag == "transposeAcc":
            i, j, *rest = pending
            return emit_acc(p.args[0], env, state, (j, i, *rest))
        if isinstance(p, dpia.ImpPrim) and p.tag in ("asVectorAcc", "asScalarAcc"):
            return emit_acc(dataclasses.replace(p, tag=VECTOR_AS[p.tag]), env, state, pending)
        return base_acc(p, env, state, pending)

    def emit(unit, target):
        text = base_emit(unit, target)
        if target != "opencl":
            head = []
            if "sqrtf(" in text or "fabsf(" in text:
                head.append("#include <math.h>")
            if re.search(r"(?<![a-z])abs\(", text):
                head.append("#include <stdlib.h>")
            if "rs_clamp(" in text:
                head.append(C_HELPERS.rstrip())
            if head:
                text = "\n".join(head) + "\n" + text
        return text

    codegen.emit_exp = emit_exp
    codegen.emit_acc = emit_acc
    codegen.emit = emit


def ensure_installed():
    if not _installed:
        install()


__all__ = ["install", "ensure_installed", "SCHEMES", "SIGNATURE_TEXT", "errors"]
