"""Loop-nest IR (LIR): the imperative DPIA of an `ImperativeUnit`, with every
functional view resolved into flat row-major index arithmetic.

This is the structured counterpart of what the reference emitter builds as
text (codegen.emit_comm / emit_exp / emit_acc, codegen.py:179-413): the same
view semantics (idx, split, join, zip/fst/snd, take and their acceptor
duals, codegen.py:199-224 and 270-286; row-major flattening,
codegen.py:157-165), plus the extension views (transpose, slide, slide2D,
padClamp, padClamp2D).  The CUDA emitter and the idiom matchers work on this
tree instead of on text, so parallel-loop mapping, shared-memory staging and
template selection are decisions over data.

Index expressions are reference `nat.Nat` terms (normalised with the unit's
divisibility assumptions, nat.py:346).  Clamped indices (padClamp) are not
polynomials, so each clamp is an opaque `nat.Var` named `__clampK` whose
meaning `min(max(inner, 0), hi)` lives in `Program.clamps`.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from ._ref import dpia, errors, nat
from ._ref import types as _types
from .types_util import scalar_ctype

EmitError = errors.EmitError
ArrayType, ScalarType, TupleType = _types.ArrayType, _types.ScalarType, _types.TupleType

# ---------------------------------------------------------------------------
# expressions (values)


@dataclass(frozen=True)
class Lit:
    text: str  # C spelling, e.g. "0.0f" or "3"
    ctype: str


@dataclass(frozen=True)
class IndexVal:
    """An integer-valued index used as data (e.g. `i` read as a value)."""

    n: object  # nat.Nat
    ctype: str = "int"


@dataclass(frozen=True)
class Load:
    buf: str
    index: object  # nat.Nat (flat)
    ctype: str
    indices: tuple = ()  # per-dimension indices before flattening (analysis only)
    vec: tuple = ()  # (w, lane var): read through asVector(w), index = base + lane, w | base


@dataclass(frozen=True)
class ScalarRef:
    name: str
    ctype: str


@dataclass(frozen=True)
class Bin:
    op: str  # + - * /
    a: object
    b: object
    ctype: str


@dataclass(frozen=True)
class Un:
    fn: str  # sqrt | rsqrt | abs
    a: object
    ctype: str


# ---------------------------------------------------------------------------
# statements


@dataclass(frozen=True)
class Store:
    buf: str
    index: object  # nat.Nat (flat)
    ctype: str
    vec: tuple = ()  # (w, lane var): written through asScalar of w-vectors, index = base + lane, w | base


@dataclass
class Assign:
    target: object  # Store | ScalarRef
    value: object


@dataclass
class Seq:
    stmts: list


@dataclass
class Alloc:
    name: str
    space: str  # "Private" | "Local" | "Global"
    ctype: str
    dims: tuple  # () for a scalar
    body: object


@dataclass
class For:
    var: str
    bound: object  # nat.Nat
    body: object


@dataclass
class ParFor:
    kind: str  # "global" | "workgroup" | "local"
    var: str
    bound: object
    body: object


@dataclass
class IfLess:
    lhs: object  # nat.Nat
    threshold: object  # nat.Nat
    then: object
    els: object


@dataclass
class DoubleBuffer:
    """Listing 11 / codegen.emit_double_buffer (codegen.py:469-504): two
    buffers, an input and an output pointer and a flag."""

    ctype: str
    size: object  # nat.Nat
    input_buf: str
    output_buf: str
    body: object


@dataclass
class Raw:
    """Verbatim statement lines (double-buffer swap / done blocks)."""

    lines: tuple


PARFOR_KIND = {"parForGlobal": "global", "parForWorkGroup": "workgroup", "parForLocal": "local"}


@dataclass
class Buffer:
    name: str
    dims: tuple  # of nat.Nat
    ctype: str
    role: str  # "input" | "output" | "alloc" | "pointer"
    space: str = "Global"
    deref: bool = False  # scalar output written through a pointer


@dataclass
class Program:
    name: str  # unit name
    nat_params: tuple  # size parameter names, in unit order
    inputs: list  # [(name, Buffer | ScalarRef)]
    output: Buffer
    body: object
    assumptions: tuple
    buffers: dict = field(default_factory=dict)
    clamps: dict = field(default_factory=dict)  # "__clampK" -> (inner Nat, hi Nat)
    names: dict = field(default_factory=dict)  # DPIA name -> C name
    peer_ranks: int = 0  # emission option: allpairs sources read from R ranks' blocks
    peer_halo: bool = False  # emission option: stencil halo rows read from the neighbours' bands


# ---------------------------------------------------------------------------
# environment bindings


@dataclass(frozen=True)
class _ArrayB:
    buf: str


@dataclass(frozen=True)
class _ScalarB:
    ref: ScalarRef


@dataclass(frozen=True)
class _IndexB:
    name: str


@dataclass(frozen=True)
class _AccB:
    buf: str | None  # array buffer name, or None for a scalar
    scalar: ScalarRef | None = None
    prefix: tuple = ()


@dataclass(frozen=True)
class _AccPhraseB:
    phrase: object
    env: dict
    prefix: tuple = ()


@dataclass(frozen=True)
class _CommB:
    stmt: object


RESERVED = {
    # C/C++ keywords and CUDA built-ins an emitted identifier must not shadow
    "auto", "break", "case", "char", "const", "continue", "default", "do", "double", "else",
    "enum", "extern", "float", "for", "goto", "if", "int", "long", "register", "return",
    "short", "signed", "sizeof", "static", "struct", "switch", "typedef", "union",
    "unsigned", "void", "volatile", "while", "bool", "true", "false", "class", "new",
    "delete", "this", "template", "typename", "namespace", "using", "private", "public",
    "protected", "operator", "friend", "virtual", "inline", "threadIdx", "blockIdx",
    "blockDim", "gridDim", "warpSize", "min", "max", "abs", "sqrt", "rsqrt", "rsqrtf",
    "sqrtf", "clamp", "ipow", "rise", "asm", "restrict", "signed", "wchar_t",
}


class Builder:
    """ImperativeUnit -> Program."""

    def __init__(self, unit):
        self.unit = unit
        self.assumptions = tuple(unit.assumptions)
        self.buffers: dict = {}
        self.clamps: dict = {}
        self.names: dict = {}
        self._used = set()
        self._clamp_cache: dict = {}
        self._vec = []  # innermost asVector / asScalarAcc being resolved: (w, lane index)

    # names ---------------------------------------------------------------
    def cname(self, name: str) -> str:
        if name in self.names:
            return self.names[name]
        out = name.replace("'", "_p")
        if out in RESERVED or out.startswith("__") or out.startswith("rs_"):
            out = out + "_"
        while out in self._used:
            out = out + "_"
        self._used.add(out)
        self.names[name] = out
        return out

    def norm(self, n):
        return nat.normalize(n, self.assumptions)

    def vec_hint(self, flat):
        """(w, lane) when the access being resolved is lane `lane` of a
        w-vector (asVector / asScalar) at a w-aligned flat index: flat =
        base + lane with every coefficient of base a multiple of w."""
        if not self._vec:
            return ()
        w, lane = self._vec[-1]
        lane = self.norm(lane)
        if not (isinstance(w, nat.Const) and w.value in (2, 4) and isinstance(lane, nat.Var)):
            return ()
        base = self.norm(flat - lane)
        if lane.name in nat.free_vars(base):
            return ()
        # w | base: every monomial has a coefficient divisible by w or a size
        # variable the unit assumes divisible by w (e.g. the row length m of
        # `row |> asVector(2)` under 2 | m)
        divisible = {num.name for num, den in self.assumptions
                     if isinstance(num, nat.Var) and isinstance(den, nat.Const) and den.value % w.value == 0}
        for mono, coeff in nat._to_poly(base, ()).items():
            if coeff % w.value and not any(isinstance(a, nat.Var) and a.name in divisible for a, _p in mono):
                return ()
        return (w.value, lane.name)

    def _with_vec(self, w, lane, fn):
        self._vec.append((w, lane))
        try:
            return fn()
        finally:
            self._vec.pop()

    def clamp(self, inner, hi):
        inner = self.norm(inner)
        hi = self.norm(hi)
        key = (inner, hi)
        var = self._clamp_cache.get(key)
        if var is None:
            var = nat.Var(f"__clamp{len(self.clamps)}")
            self.clamps[var.name] = (inner, hi)
            self._clamp_cache[key] = var
        return var

    # top level -----------------------------------------------------------
    def build(self) -> Program:
        unit = self.unit
        for p in unit.nat_params:
            self._used.add(p)
            self.names[p] = p
        env = {}
        inputs = []
        for var, dtype in unit.inputs:
            name = self.cname(var.name)
            if isinstance(dtype, ScalarType):
                ref = ScalarRef(name, scalar_ctype(dtype))
                env[var.uid] = _ScalarB(ref)
                inputs.append((name, ref))
            else:
                dims, elem = _shape(dtype)
                buf = Buffer(name, dims, scalar_ctype(elem), "input")
                self.buffers[name] = buf
                env[var.uid] = _ArrayB(name)
                inputs.append((name, buf))
        dims, elem = _shape(unit.output_type)
        oname = self.cname(unit.output.name)
        out = Buffer(oname, dims if dims else (nat.Const(1),), scalar_ctype(elem), "output", deref=not dims)
        self.buffers[oname] = out
        env[unit.output.uid] = _AccB(oname)
        body = self.comm(unit.body, env)
        return Program(
            name=unit.name,
            nat_params=tuple(unit.nat_params),
            inputs=inputs,
            output=out,
            body=body,
            assumptions=self.assumptions,
            buffers=self.buffers,
            clamps=self.clamps,
            names=self.names,
        )

    # indices ---------------------------------------------------------------
    def flat(self, buf: Buffer, indices):
        if buf.deref:
            if indices:
                raise EmitError("indexing into a scalar output")
            return nat.Const(0)
        if len(indices) != len(buf.dims):
            raise EmitError(
                f"dimension mismatch on {buf.name}: {len(indices)} indices for {len(buf.dims)} dims"
            )
        flat = indices[0]
        for dim, ix in zip(buf.dims[1:], indices[1:]):
            flat = flat * dim + ix
        return self.norm(flat)

    def index_of(self, p, env):
        if isinstance(p, dpia.PhraseVar):
            b = env.get(p.uid)
            if isinstance(b, _IndexB):
                return nat.Var(b.name)
            raise EmitError(f"index expression is not a loop variable: {p.name}")
        if isinstance(p, dpia.PhraseLiteral) and isinstance(p.value, int) and not isinstance(p.value, bool):
            return nat.Const(p.value)
        raise EmitError("unsupported index expression form")

    # reads -------------------------------------------------------------------
    def lookup(self, p, env):
        if isinstance(p, dpia.PhraseVar):
            b = env.get(p.uid)
            if b is None:
                raise EmitError(f"unbound name {p.name!r} during emission")
            return b
        if isinstance(p, dpia.PhraseProj):
            path = []
            q = p
            while isinstance(q, dpia.PhraseProj):
                path.append(q.index)
                q = q.pair
            if isinstance(q, dpia.PhraseVar):
                value = env.get(q.uid)
                for index in reversed(path):
                    if not isinstance(value, tuple):
                        return None
                    value = value[0] if index == 1 else value[1]
                return value
        return None

    def exp(self, p, env, pending=(), projs=()):
        if isinstance(p, (dpia.PhraseVar, dpia.PhraseProj)):
            b = self.lookup(p, env)
            if isinstance(b, _ScalarB):
                if pending or projs:
                    raise EmitError(f"scalar {b.ref.name} used with indices")
                return b.ref
            if isinstance(b, _IndexB):
                if pending or projs:
                    raise EmitError("index used with indices")
                return IndexVal(nat.Var(b.name))
            if isinstance(b, _ArrayB):
                if projs:
                    raise EmitError("tuple projection reached array memory; zips must stay views")
                buf = self.buffers[b.buf]
                idx = tuple(self.norm(i) for i in pending) if not buf.deref else ()
                flat = self.flat(buf, list(pending))
                return Load(buf.name, flat, buf.ctype, idx, self.vec_hint(flat) if not buf.deref else ())
            raise EmitError(f"cannot read {p!r}")
        if isinstance(p, dpia.PhraseLiteral):
            return Lit(p.text, _lit_ctype(p))
        if isinstance(p, dpia.FunPrim):
            tag = p.tag
            ta = p.type_args
            a0 = p.args[0] if p.args else None
            if tag == "idx":
                i = self.index_of(p.args[0], env)
                return self.exp(p.args[1], env, (i,) + tuple(pending), projs)
            if tag == "split":
                chunk = ta[0]
                c, j, *rest = pending
                return self.exp(a0, env, (c * chunk + j, *rest), projs)
            if tag == "asVector":  # split(w), and the access is lane j of a w-vector
                chunk = ta[0]
                c, j, *rest = pending
                return self._with_vec(chunk, j, lambda: self.exp(a0, env, (c * chunk + j, *rest), projs))
            if tag == "asScalar":  # join: the flat index's vector lane is f % w
                inner = ta[1]
                f, *rest = pending
                return self.exp(a0, env, (nat.Div(f, inner), nat.Mod(f, inner), *rest), projs)
            if tag == "join":
                inner = ta[1]
                f, *rest = pending
                return self.exp(a0, env, (nat.Div(f, inner), nat.Mod(f, inner), *rest), projs)
            if tag == "take":
                return self.exp(a0, env, pending, projs)
            if tag == "zip":
                if not projs:
                    raise EmitError("zip read without a projection")
                side = projs[-1]
                return self.exp(p.args[0] if side == 1 else p.args[1], env, pending, projs[:-1])
            if tag == "fst":
                return self.exp(a0, env, pending, tuple(projs) + (1,))
            if tag == "snd":
                return self.exp(a0, env, pending, tuple(projs) + (2,))
            if tag == "transpose":
                i, j, *rest = pending
                return self.exp(a0, env, (j, i, *rest), projs)
            if tag == "slide":
                sz, sp = ta[0], ta[1]
                i, a, *rest = pending
                return self.exp(a0, env, (i * sp + a, *rest), projs)
            if tag == "slide2D":
                sz, sp = ta[0], ta[1]
                i, j, a, b, *rest = pending
                return self.exp(a0, env, (i * sp + a, j * sp + b, *rest), projs)
            if tag == "padClamp":
                l, _r, n = ta[0], ta[1], ta[2]
                i, *rest = pending
                return self.exp(a0, env, (self.clamp(i - l, n - nat.Const(1)), *rest), projs)
            if tag == "padClamp2D":
                l, _r, n, m = ta[0], ta[1], ta[2], ta[3]
                i, j, *rest = pending
                ci = self.clamp(i - l, n - nat.Const(1))
                cj = self.clamp(j - l, m - nat.Const(1))
                return self.exp(a0, env, (ci, cj, *rest), projs)
            if tag in ("add", "sub", "mul", "div"):
                if pending or projs:
                    raise EmitError("indexed arithmetic value")
                a = self.exp(p.args[0], env)
                b = self.exp(p.args[1], env)
                op = {"add": "+", "sub": "-", "mul": "*", "div": "/"}[tag]
                return Bin(op, a, b, _value_ctype(a, b))
            if tag in ("sqrt", "rsqrt"):
                if pending or projs:
                    raise EmitError("indexed arithmetic value")
                a = self.exp(a0, env)
                return Un(tag, a, "float")
            if tag == "abs":
                if pending or projs:
                    raise EmitError("indexed arithmetic value")
                a = self.exp(a0, env)
                return Un(tag, a, getattr(a, "ctype", "float"))
        raise EmitError(f"no emission for expression {getattr(p, 'tag', type(p).__name__)}")

    # writes ------------------------------------------------------------------
    def acc(self, p, env, pending=()):
        if isinstance(p, (dpia.PhraseVar, dpia.PhraseProj)):
            b = self.lookup(p, env)
            if isinstance(b, _AccPhraseB):
                return self.acc(b.phrase, b.env, tuple(b.prefix) + tuple(pending))
            if isinstance(b, _AccB):
                idx = list(b.prefix) + list(pending)
                if b.scalar is not None:
                    if idx:
                        raise EmitError(f"indexing into scalar {b.scalar.name}")
                    return b.scalar
                buf = self.buffers[b.buf]
                flat = self.flat(buf, idx)
                return Store(buf.name, flat, buf.ctype, self.vec_hint(flat))
            raise EmitError(f"cannot write through {p!r}")
        if isinstance(p, dpia.ImpPrim):
            tag = p.tag
            ta = p.type_args
            if tag == "idxAcc":
                i = self.index_of(p.args[0], env)
                return self.acc(p.args[1], env, (i,) + tuple(pending))
            if tag == "joinAcc":
                inner = ta[1]
                a, b, *rest = pending
                return self.acc(p.args[0], env, (a * inner + b, *rest))
            if tag == "asScalarAcc":  # joinAcc, and the write is lane b of a w-vector
                inner = ta[1]
                a, b, *rest = pending
                return self._with_vec(inner, b, lambda: self.acc(p.args[0], env, (a * inner + b, *rest)))
            if tag == "asVectorAcc":  # splitAcc
                chunk = ta[0]
                f, *rest = pending
                return self.acc(p.args[0], env, (nat.Div(f, chunk), nat.Mod(f, chunk), *rest))
            if tag == "splitAcc":
                chunk = ta[0]
                f, *rest = pending
                return self.acc(p.args[0], env, (nat.Div(f, chunk), nat.Mod(f, chunk), *rest))
            if tag == "takeAcc":
                return self.acc(p.args[0], env, pending)
            if tag == "transposeAcc":
                i, j, *rest = pending
                return self.acc(p.args[0], env, (j, i, *rest))
            if tag in ("zipAcc1", "zipAcc2"):
                raise EmitError("tuple-typed memory has no flat layout; keep zips as views")
        raise EmitError(f"no emission for acceptor {getattr(p, 'tag', type(p).__name__)}")

    # commands ----------------------------------------------------------------
    def comm(self, p, env):
        if isinstance(p, (dpia.PhraseVar, dpia.PhraseProj)):
            b = self.lookup(p, env)
            if isinstance(b, _CommB):
                return b.stmt
            raise EmitError("expected a command")
        if not isinstance(p, dpia.ImpPrim):
            raise EmitError(f"cannot emit {p!r} as a statement")
        tag = p.tag
        if tag == "seq":
            a = self.comm(p.args[0], env)
            b = self.comm(p.args[1], env)
            return Seq(_flatten_seq([a, b]))
        if tag == "assign":
            return Assign(self.acc(p.args[0], env), self.exp(p.args[1], env))
        if tag == "new":
            space, dtype = p.type_args
            body = p.args[0]
            name = self.cname(body.param.name)
            if isinstance(dtype, ScalarType):
                ref = ScalarRef(name, scalar_ctype(dtype))
                pair = (_ScalarB(ref), _AccB(None, ref))
                return Alloc(name, space.value, ref.ctype, (), self.comm(body.body, {**env, body.param.uid: pair}))
            dims, elem = _shape(dtype)
            buf = Buffer(name, dims, scalar_ctype(elem), "alloc", space=space.value)
            self.buffers[name] = buf
            pair = (_ArrayB(name), _AccB(name))
            return Alloc(name, space.value, buf.ctype, dims, self.comm(body.body, {**env, body.param.uid: pair}))
        if tag == "for":
            bound = self.norm(p.type_args[0])
            body = p.args[0]
            name = self.cname(body.param.name)
            return For(name, bound, self.comm(body.body, {**env, body.param.uid: _IndexB(name)}))
        if tag in PARFOR_KIND:
            bound = self.norm(p.type_args[0])
            out = p.args[0]
            lam = p.args[1]
            ivar, inner = lam.param, lam.body
            ovar = inner.param
            name = self.cname(ivar.name)
            slot = _AccPhraseB(out, env, (nat.Var(name),))
            inner_env = {**env, ivar.uid: _IndexB(name), ovar.uid: slot}
            return ParFor(PARFOR_KIND[tag], name, bound, self.comm(inner.body, inner_env))
        if tag == "ifLess":
            threshold = self.norm(p.type_args[1])
            lhs = self.index_of(p.args[0], env)
            return IfLess(lhs, threshold, self.comm(p.args[1], env), self.comm(p.args[2], env))
        if tag == "newDoubleBuffer":
            return self._double_buffer(p, env)
        raise EmitError(f"no emission for command {tag!r}")

    def _whole_array(self, p, env, what):
        b = self.lookup(p, env) if isinstance(p, (dpia.PhraseVar, dpia.PhraseProj)) else None
        if isinstance(b, _AccB) and not b.prefix and b.buf is not None:
            return b.buf
        if isinstance(b, _ArrayB):
            return b.buf
        raise EmitError(f"{what} must be a whole array, not a view")

    def _double_buffer(self, p, env):
        dtype, buf_size, _out_len, _in_len = p.type_args
        input_p, output_p, body = p.args
        elem = dtype if isinstance(dtype, ScalarType) else _shape(dtype)[1]
        ctype = scalar_ctype(elem)
        size = self.norm(buf_size)
        in_buf = self._whole_array(input_p, env, "double-buffer input")
        out_buf = self._whole_array(output_p, env, "double-buffer output")
        for name in ("in_ptr", "out_ptr"):
            self.buffers[name] = Buffer(name, (size,), ctype, "pointer")
        swap = Raw((
            "in_ptr = flag ? buffer1 : buffer2;",
            "out_ptr = flag ? buffer2 : buffer1;",
            "flag = flag ^ 1;",
        ))
        done = Raw(("in_ptr = flag ? buffer1 : buffer2;", f"out_ptr = {out_buf};"))
        components = (((_AccB("out_ptr"), _ArrayB("in_ptr")), _CommB(swap)), _CommB(done))
        inner = self.comm(body.body, {**env, body.param.uid: components})
        return DoubleBuffer(ctype, size, in_buf, out_buf, inner)


def _shape(dt):
    dims = []
    while isinstance(dt, ArrayType):
        dims.append(dt.size)
        dt = dt.elem
    if isinstance(dt, TupleType):
        raise EmitError("tuple-typed memory has no flat layout; keep zips as views")
    return tuple(dims), dt


def _lit_ctype(p):
    if isinstance(p.value, bool) or isinstance(p.value, int):
        return "int"
    return "float"


def _value_ctype(a, b):
    ca = getattr(a, "ctype", "float")
    cb = getattr(b, "ctype", "float")
    return "float" if "float" in (ca, cb) else "int"


def _flatten_seq(stmts):
    out = []
    for s in stmts:
        if isinstance(s, Seq):
            out.extend(_flatten_seq(s.stmts))
        else:
            out.append(s)
    return out


def build(unit) -> Program:
    return Builder(unit).build()


# ---------------------------------------------------------------------------
# traversal helpers used by the emitter and the idiom matchers


def walk(stmt):
    """Pre-order traversal of statements."""
    yield stmt
    for c in children(stmt):
        yield from walk(c)


def children(stmt):
    if isinstance(stmt, Seq):
        return list(stmt.stmts)
    if isinstance(stmt, (Alloc, For, ParFor, DoubleBuffer)):
        return [stmt.body]
    if isinstance(stmt, IfLess):
        return [stmt.then, stmt.els]
    return []


def expr_loads(e):
    """Every Load inside a value expression."""
    if isinstance(e, Load):
        yield e
    elif isinstance(e, Bin):
        yield from expr_loads(e.a)
        yield from expr_loads(e.b)
    elif isinstance(e, Un):
        yield from expr_loads(e.a)


def expr_scalars(e):
    if isinstance(e, ScalarRef):
        yield e
    elif isinstance(e, Bin):
        yield from expr_scalars(e.a)
        yield from expr_scalars(e.b)
    elif isinstance(e, Un):
        yield from expr_scalars(e.a)


def stmt_exprs(stmt):
    """(target, value) pairs of all assignments below `stmt`."""
    for s in walk(stmt):
        if isinstance(s, Assign):
            yield s.target, s.value


def nat_vars(n) -> set:
    return nat.free_vars(n)
