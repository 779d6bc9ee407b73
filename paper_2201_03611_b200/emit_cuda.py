"""ImperativeUnit -> CUDA C++ for sm_100a (the `sm100a` emit target).

Replaces the reference back end `codegen.emit(unit, target)` (codegen.py:451)
for GPUs.  The reference's OpenCL mapping has three constructs that are
invalid on a real GPU (SURVEY.md §8 a, list after the table); this emitter
maps the same imperative phrases to a valid CUDA execution:

* perfectly nested `parForGlobal` chains collapse into one grid-stride loop
  over their product (instead of all loops sharing `get_global_id(0)`);
* `parForWorkGroup` is a block-strided loop whose body runs block-uniformly:
  `parForLocal` becomes a thread-strided loop followed by `__syncthreads()`,
  `new(Local)` (and per-work-group `new(Private)` arrays) become `__shared__`
  arrays, and sequential statements with memory effects run on thread 0
  followed by a barrier;
* `toMem(Global)` between parallel stages splits the unit into one kernel
  per stage, with the temporary allocated by the runtime.

Stages whose loop nest matches a hand-written template (`idioms.py`) are
emitted as an instantiation of that template; the generic kernel for the
same stage is kept in the text as the fallback when a template's run-time
precondition (alignment, divisibility) does not hold.

Sizes become template parameters, instantiated at NVRTC time with the
run-time sizes (SURVEY.md §8 b "Kernel ABI"), so array extents and index
arithmetic are compile-time constants.  The text is deterministic (byte
stable for a given unit, like codegen.emit, test_codegen.py:71-74) and
carries its launch plan as a JSON comment, so `run_cuda(code, unit, ...)`
needs nothing but the text — the same contract as `cexec.run_emitted`.

Arithmetic: with `exact=True` (default) every f32 operation is rendered with
the round-to-nearest intrinsics (`__fadd_rn`, `__fmul_rn`, ...), which the
compiler never contracts into FMAs, so a kernel that preserves the program's
evaluation order is bit-exact with the reference's sequential fp32
semantics (interpreter.py:161-169).
"""

from __future__ import annotations

import json
import os
import warnings
from dataclasses import dataclass, field

from . import lir
from ._ref import codegen, errors, nat

EmitError = errors.EmitError

TARGET = "sm100a"
PLAN_TAG = "// @plan "

DEFAULT_BLOCK = 256

# ---------------------------------------------------------------------------
# rendering of sizes / indices


def _has_pow(n) -> bool:
    if isinstance(n, nat.Pow):
        return True
    if isinstance(n, nat.Sum):
        return any(_has_pow(t) for t in n.terms)
    if isinstance(n, nat.Product):
        return any(_has_pow(f) for f in n.factors)
    if isinstance(n, (nat.Div, nat.Mod)):
        return _has_pow(n.num) or _has_pow(n.den)
    return False


class NatRenderer:
    """Nat -> C (or Python) integer expression text.

    Plain C index text is the reference emitter's own rendering
    (codegen._render, codegen.py:80-110: the same normal form, precedence
    and negation handling), so emitted indices read exactly like the
    reference's.  This class adds what the reference has no notion of:
    clamped (padClamp) index atoms -> rs_clamp(...), renamed variables,
    `ipow` spelled rs_ipow, and the Python spelling (// and **) of launch
    expressions evaluated by the planner."""

    def __init__(self, clamps=None, py=False, names=None):
        self.clamps = clamps or {}
        self.py = py
        self.names = names or {}

    def __call__(self, n, prec=0):
        return self.render(n, prec)

    def render(self, n, prec=0):
        if not self.py and not _has_pow(n) and not (nat.free_vars(n) & (set(self.clamps) | set(self.names))):
            return codegen._render(n, codegen._State(TARGET, ()), prec)
        return self._render(n, prec)

    def _render(self, n, prec=0):
        if isinstance(n, nat.Const):
            return str(n.value) if n.value >= 0 else f"(-{-n.value})"
        if isinstance(n, nat.Var):
            if n.name in self.clamps:
                inner, hi = self.clamps[n.name]
                if self.py:
                    raise EmitError("clamped index in a launch expression")
                return f"rs_clamp({self.render(inner)}, {self.render(hi)})"
            return self.names.get(n.name, n.name)
        if isinstance(n, nat.Sum):
            parts = []
            terms = [nat._strip_negation(t) for t in n.terms]
            terms = [t for t in terms if not t[0]] + [t for t in terms if t[0]]
            for k, (neg, body) in enumerate(terms):
                s = self.render(body, 1)
                if k == 0:
                    parts.append(f"-{s}" if neg else s)
                else:
                    parts.append((" - " if neg else " + ") + s)
            text = "".join(parts)
            return f"({text})" if prec > 1 else text
        if isinstance(n, nat.Product):
            text = " * ".join(self.render(f, 2) for f in n.factors)
            return f"({text})" if prec > 2 else text
        if isinstance(n, nat.Div):
            op = " // " if self.py else " / "
            text = f"{self.render(n.num, 3)}{op}{self.render(n.den, 3)}"
            return f"({text})" if prec >= 2 else text
        if isinstance(n, nat.Mod):
            text = f"{self.render(n.num, 3)} % {self.render(n.den, 3)}"
            return f"({text})" if prec >= 2 else text
        if isinstance(n, nat.Pow):
            if self.py:
                return f"({self.render(n.base, 3)} ** {self.render(n.exp, 3)})"
            return f"rs_ipow({self.render(n.base)}, {self.render(n.exp)})"
        raise EmitError(f"cannot render size expression {n!r}")


def py_expr(n) -> str:
    """Python text of a size expression (evaluated by the launch planner)."""
    return NatRenderer(py=True)(nat.normalize(n))


def eval_py(expr: str, nats: dict) -> int:
    return int(eval(expr, {"__builtins__": {}}, dict(nats)))  # noqa: S307 - self-generated text


# ---------------------------------------------------------------------------
# rendering of values


class ValueRenderer:
    def __init__(self, prog: lir.Program, exact=True, load_hook=None):
        self.prog = prog
        self.exact = exact
        self.nat = NatRenderer(prog.clamps)
        self.load_hook = load_hook  # optional (Load) -> str override (smem staging)

    def __call__(self, e):
        return self.val(e)

    def val(self, e):
        if isinstance(e, lir.Lit):
            return e.text
        if isinstance(e, lir.IndexVal):
            return f"({self.nat(e.n)})"
        if isinstance(e, lir.ScalarRef):
            return e.name
        if isinstance(e, lir.Load):
            if self.load_hook is not None:
                out = self.load_hook(e)
                if out is not None:
                    return out
            return f"{e.buf}[{self.nat(e.index)}]"
        if isinstance(e, lir.Bin):
            a, b = self.val(e.a), self.val(e.b)
            if e.ctype == "float" and self.exact:
                fn = {"+": "__fadd_rn", "-": "__fsub_rn", "*": "__fmul_rn", "/": "__fdiv_rn"}[e.op]
                return f"{fn}({a}, {b})"
            return f"({a} {e.op} {b})"
        if isinstance(e, lir.Un):
            a = self.val(e.a)
            if e.fn == "sqrt":
                return f"__fsqrt_rn({a})" if self.exact else f"sqrtf({a})"
            if e.fn == "rsqrt":
                return f"rs_rsqrt_exact({a})" if self.exact else f"rs_rsqrt_fast({a})"
            if e.fn == "abs":
                return f"fabsf({a})" if e.ctype == "float" else f"abs({a})"
        raise EmitError(f"cannot render value {e!r}")

    def target(self, t):
        if isinstance(t, lir.ScalarRef):
            return t.name
        if isinstance(t, lir.Store):
            return f"{t.buf}[{self.nat(t.index)}]"
        raise EmitError(f"cannot render target {t!r}")


# ---------------------------------------------------------------------------
# stage analysis


def contains_parfor(stmt) -> bool:
    return any(isinstance(s, lir.ParFor) for s in lir.walk(stmt))


def collapse_global_chain(stmt):
    """ParFor(global) perfectly nested chain -> ([(var, bound)...], body)."""
    loops = []
    while isinstance(stmt, lir.ParFor) and stmt.kind == "global":
        loops.append((stmt.var, stmt.bound))
        stmt = stmt.body
    return loops, stmt


@dataclass
class Stage:
    kind: str  # "grid" | "workgroup" | "block" | "serial"
    stmt: object
    index: int = 0


@dataclass
class Temp:
    name: str
    ctype: str
    dims: tuple


def split_stages(body, prog):
    """Top-level statements -> kernel stages; Global (and parallel-shared)
    temporaries become runtime-allocated buffers."""
    temps = []
    stages = []

    def visit(s):
        if isinstance(s, lir.Alloc) and s.dims and (s.space == "Global" or contains_parfor(s.body)):
            temps.append(Temp(s.name, s.ctype, s.dims))
            prog.buffers[s.name].space = "Global"
            visit(s.body)
            return
        if isinstance(s, lir.Seq):
            for c in s.stmts:
                visit(c)
            return
        if isinstance(s, lir.ParFor) and s.kind == "global":
            stages.append(Stage("grid", s))
        elif isinstance(s, lir.ParFor) and s.kind == "workgroup":
            stages.append(Stage("workgroup", s))
        elif contains_parfor(s):
            stages.append(Stage("block", s))
        else:
            stages.append(Stage("serial", s))

    visit(body)
    merged = []
    for st in stages:  # adjacent serial statements share one kernel
        if merged and st.kind == "serial" and merged[-1].kind == "serial":
            merged[-1] = Stage("serial", lir.Seq([merged[-1].stmt, st.stmt]))
        else:
            merged.append(st)
    for k, st in enumerate(merged):
        st.index = k
    return merged, temps


# ---------------------------------------------------------------------------
# kernel text


@dataclass
class KernelText:
    name: str
    text: str
    plan: dict


@dataclass
class CudaCode:
    text: str
    plan: dict
    program: lir.Program = field(repr=False, default=None)


def _map_value(e, load_fn, sub):
    """Rebuild a value with `load_fn` applied to its loads and the index
    substitution `sub` applied to every index."""
    if isinstance(e, lir.Load):
        return load_fn(e)
    if isinstance(e, lir.IndexVal):
        return lir.IndexVal(nat.normalize(nat.substitute(e.n, sub)), e.ctype)
    if isinstance(e, lir.Bin):
        return lir.Bin(e.op, _map_value(e.a, load_fn, sub), _map_value(e.b, load_fn, sub), e.ctype)
    if isinstance(e, lir.Un):
        return lir.Un(e.fn, _map_value(e.a, load_fn, sub), e.ctype)
    return e


class GenericKernel:
    """One stage -> one kernel with the generic GPU mapping.

    `vectorize=True`: a constant loop over the w = 2 / 4 lanes of a vector
    (asVector / asScalar views: lir.Load.vec / Store.vec) reads its lanes
    with one float2 / float4 load and writes them with one vector store —
    Shine's vector types as float4 pointers.  The
    caller keeps the scalar kernel as the fallback for buffers that are not
    16-byte aligned."""

    def __init__(self, prog: lir.Program, stage: Stage, name: str, temps, exact=True, vectorize=False):
        self.prog = prog
        self.stage = stage
        self.name = name
        self.temps = temps
        self.r = ValueRenderer(prog, exact)
        self.nat = self.r.nat
        self.shared_decls = []
        self.shared_names = set()
        self.smem_bytes = []  # py size expressions of static shared arrays
        self.vectorize = vectorize
        self.vector_accesses = 0  # vector loads + stores emitted

    def _vector_for(self, s, ind):
        """The lanes loop of a vector: one vector load per (buffer, base),
        the w lanes unrolled, one vector store per written vector; None when
        the loop does not qualify."""
        w, v = s.bound.value, s.var
        body = s.body.stmts if isinstance(s.body, lir.Seq) else [s.body]
        if not all(isinstance(x, lir.Assign) for x in body):
            return None
        written = {x.target.buf for x in body if isinstance(x.target, lir.Store)}
        read = {ld.buf for x in body for ld in lir.expr_loads(x.value)}

        def base_of(ix):
            return nat.normalize(ix - nat.Var(v))

        loads, stores = {}, {}
        for x in body:
            for ld in lir.expr_loads(x.value):
                if ld.vec == (w, v) and ld.ctype == "float" and ld.buf not in written:
                    loads.setdefault((ld.buf, base_of(ld.index)), f"rs_vl{len(loads)}")
        scalar_written = {x.target.buf for x in body
                          if isinstance(x.target, lir.Store) and not (x.target.vec == (w, v) and x.target.ctype == "float")}
        for x in body:
            t = x.target
            if (isinstance(t, lir.Store) and t.vec == (w, v) and t.ctype == "float" and t.buf not in read
                    and t.buf not in scalar_written):
                key = (t.buf, base_of(t.index))
                if key in stores:
                    return None  # a lane written twice: keep the scalar order
                stores[key] = f"rs_vs{len(stores)}"
        if not loads and not stores:
            return None
        vt = "float4" if w == 4 else "float2"
        p = "  " * ind
        out = [f"{p}{{  // the {w} lanes of a vector: {vt} accesses"]
        for (buf, base), nm in loads.items():
            out.append(f"{p}  const {vt} {nm} = *reinterpret_cast<const {vt}*>({buf} + ({self.nat(base)}));")
        for (buf, base), nm in stores.items():
            out.append(f"{p}  {vt} {nm};")
        for k in range(w):
            comp = "xyzw"[k]
            sub = {v: nat.Const(k)}

            def load_fn(ld, comp=comp, sub=sub):
                key = (ld.buf, base_of(ld.index))
                if ld.vec == (w, v) and key in loads:
                    return lir.ScalarRef(f"{loads[key]}.{comp}", ld.ctype)
                return lir.Load(ld.buf, nat.normalize(nat.substitute(ld.index, sub)), ld.ctype)

            lane = []
            for x in body:
                t = x.target
                if isinstance(t, lir.Store):
                    key = (t.buf, base_of(t.index))
                    if t.vec == (w, v) and key in stores:
                        t = lir.ScalarRef(f"{stores[key]}.{comp}", t.ctype)
                    else:
                        t = lir.Store(t.buf, nat.normalize(nat.substitute(t.index, sub)), t.ctype)
                lane.append(lir.Assign(t, _map_value(x.value, load_fn, sub)))
            out += self.thread(lir.Seq(lane), ind + 1)
        for (buf, base), nm in stores.items():
            out.append(f"{p}  *reinterpret_cast<{vt}*>({buf} + ({self.nat(base)})) = {nm};")
        out.append(f"{p}}}")
        self.vector_accesses += len(loads) + len(stores)
        return out

    # helpers -------------------------------------------------------------
    def _size_c(self, dims):
        size = dims[0]
        for d in dims[1:]:
            size = size * d
        return self.nat(nat.normalize(size))

    def _declare_shared(self, name, ctype, dims):
        if name in self.shared_names:
            return
        self.shared_names.add(name)
        if dims:
            self.shared_decls.append(f"__shared__ {ctype} {name}[{self._size_c(dims)}];")
            size = dims[0]
            for d in dims[1:]:
                size = size * d
            self.smem_bytes.append(f"4 * ({py_expr(size)})")
        else:
            self.shared_decls.append(f"__shared__ {ctype} {name};")
            self.smem_bytes.append("4")

    # thread-level code (sequential semantics inside one thread) -----------
    def thread(self, s, ind):
        p = "  " * ind
        if isinstance(s, lir.Seq):
            out = []
            for c in s.stmts:
                out += self.thread(c, ind)
            return out
        if isinstance(s, lir.Assign):
            return [f"{p}{self.r.target(s.target)} = {self.r(s.value)};"]
        if isinstance(s, lir.Alloc):
            if s.dims:
                decl = f"{p}{s.ctype} {s.name}[{self._size_c(s.dims)}];"
            else:
                decl = f"{p}{s.ctype} {s.name};"
            return [decl] + self.thread(s.body, ind)
        if (self.vectorize and isinstance(s, lir.For) and isinstance(s.bound, nat.Const)
                and s.bound.value in (2, 4)):
            out = self._vector_for(s, ind)
            if out is not None:
                return out
        if isinstance(s, (lir.For, lir.ParFor)):
            head = f"{p}for (int {s.var} = 0; {s.var} < {self.nat(s.bound)}; {s.var} += 1) {{"
            pre = []
            if isinstance(s.bound, nat.Const) and s.bound.value <= 16:
                pre = ["#pragma unroll"]  # small windows: constant register indices
            return pre + [head] + self.thread(s.body, ind + 1) + [f"{p}}}"]
        if isinstance(s, lir.IfLess):
            return (
                [f"{p}if ({self.nat(s.lhs)} < {self.nat(s.threshold)}) {{"]
                + self.thread(s.then, ind + 1)
                + [f"{p}}} else {{"]
                + self.thread(s.els, ind + 1)
                + [f"{p}}}"]
            )
        if isinstance(s, lir.Raw):
            return [p + line for line in s.lines]
        if isinstance(s, lir.DoubleBuffer):
            size = self.nat(s.size)
            c = s.ctype
            return [
                f"{p}{c} buffer1[{size}]; {c} buffer2[{size}];",
                f"{p}const {c}* in_ptr = {s.input_buf}; {c}* out_ptr = buffer1;",
                f"{p}unsigned char flag = 1;",
            ] + self.thread(s.body, ind)
        raise EmitError(f"cannot emit statement {s!r}")

    # block-uniform code (all threads of the block, with barriers) ---------
    def block(self, s, ind):
        p = "  " * ind
        if isinstance(s, lir.Seq):
            out = []
            for c in s.stmts:
                out += self.block(c, ind)
            return out
        if not contains_parfor(s):
            if isinstance(s, lir.Alloc):
                self._declare_shared(s.name, s.ctype, s.dims)
                return self.block(s.body, ind)
            # sequential statement: thread 0 performs it, everyone waits
            return [f"{p}if (threadIdx.x == 0) {{"] + self.thread_shared(s, ind + 1) + [
                f"{p}}}", f"{p}__syncthreads();"]
        if isinstance(s, lir.ParFor):
            head = (f"{p}for (int {s.var} = threadIdx.x; {s.var} < {self.nat(s.bound)}; "
                    f"{s.var} += blockDim.x) {{")
            return [head] + self.thread(s.body, ind + 1) + [f"{p}}}", f"{p}__syncthreads();"]
        if isinstance(s, lir.Alloc):
            self._declare_shared(s.name, s.ctype, s.dims)
            return self.block(s.body, ind)
        if isinstance(s, lir.For):
            head = f"{p}for (int {s.var} = 0; {s.var} < {self.nat(s.bound)}; {s.var} += 1) {{"
            return [head] + self.block(s.body, ind + 1) + [f"{p}}}"]
        if isinstance(s, lir.IfLess):
            return (
                [f"{p}if ({self.nat(s.lhs)} < {self.nat(s.threshold)}) {{"]
                + self.block(s.then, ind + 1)
                + [f"{p}}} else {{"]
                + self.block(s.els, ind + 1)
                + [f"{p}}}"]
            )
        if isinstance(s, lir.DoubleBuffer):
            size = self.nat(s.size)
            c = s.ctype
            self.shared_decls += [
                f"__shared__ {c} buffer1[{size}]; __shared__ {c} buffer2[{size}];",
                f"__shared__ const {c}* in_ptr; __shared__ {c}* out_ptr;",
                "__shared__ unsigned char flag;",
            ]
            self.smem_bytes.append(f"8 * ({py_expr(s.size)})")
            return [
                f"{p}if (threadIdx.x == 0) {{",
                f"{p}  in_ptr = {s.input_buf}; out_ptr = buffer1; flag = 1;",
                f"{p}}}",
                f"{p}__syncthreads();",
            ] + self.block(s.body, ind)
        raise EmitError(f"cannot emit statement {s!r} at block level")

    def thread_shared(self, s, ind):
        """Sequential code run by thread 0 where block-level allocations are
        shared variables (already declared)."""
        return self.thread(s, ind)

    # whole kernel ---------------------------------------------------------
    def emit(self) -> KernelText:
        st = self.stage
        body = []
        plan = {"name": self.name, "kind": st.kind}
        if st.kind == "grid":
            loops, inner = collapse_global_chain(st.stmt)
            total = nat.Const(1)
            for _, b in loops:
                total = total * b
            total = nat.normalize(total, self.prog.assumptions)
            body.append(f"  const int rs_total = {self.nat(total)};")
            body.append("  for (int rs_f = blockIdx.x * blockDim.x + threadIdx.x; rs_f < rs_total; "
                        "rs_f += gridDim.x * blockDim.x) {")
            rest = "rs_f"
            for k, (var, bound) in enumerate(loops):
                if k == len(loops) - 1:
                    body.append(f"    const int {var} = {rest};")
                else:
                    inner_size = nat.Const(1)
                    for _, b in loops[k + 1:]:
                        inner_size = inner_size * b
                    size_c = self.nat(nat.normalize(inner_size, self.prog.assumptions), 2)
                    body.append(f"    const int {var} = {rest} / {size_c};")
                    body.append(f"    const int rs_r{k} = {rest} % {size_c};")
                    rest = f"rs_r{k}"
            body += self.thread(inner, 2)
            body.append("  }")
            plan.update(total=py_expr(total), block=DEFAULT_BLOCK)
        elif st.kind == "workgroup":
            wg = st.stmt
            body.append(f"  for (int {wg.var} = blockIdx.x; {wg.var} < {self.nat(wg.bound)}; "
                        f"{wg.var} += gridDim.x) {{")
            body += self.block(wg.body, 2)
            body.append("    __syncthreads();")
            body.append("  }")
            locals_ = [s.bound for s in lir.walk(wg.body) if isinstance(s, lir.ParFor)]
            plan.update(total=py_expr(wg.bound), block=DEFAULT_BLOCK,
                        local_bounds=[py_expr(b) for b in locals_])
        elif st.kind == "block":
            body += self.block(st.stmt, 1)
            plan.update(total="1", block=DEFAULT_BLOCK)
        else:  # serial
            body += self.thread(st.stmt, 1)
            plan.update(total="1", block=1)
        plan["smem_static"] = " + ".join(self.smem_bytes) if self.smem_bytes else "0"
        head = kernel_head(self.prog, self.name, self.temps,
                           launch_bounds=plan["block"] if st.kind != "serial" else 1)
        lines = head + ["  " + d for d in self.shared_decls] + body + ["}"]
        return KernelText(self.name, "\n".join(lines) + "\n", plan)


def kernel_params(prog: lir.Program, temps):
    params = [f"{prog.output.ctype}* __restrict__ {prog.output.name}"]
    for name, b in prog.inputs:
        if isinstance(b, lir.ScalarRef):
            params.append(f"{b.ctype} {name}")
        else:
            params.append(f"const {b.ctype}* __restrict__ {name}")
    for t in temps:
        params.append(f"{t.ctype}* __restrict__ {t.name}")
    return params


def template_line(prog: lir.Program):
    if not prog.nat_params:
        return []
    return ["template <" + ", ".join(f"int {n}" for n in prog.nat_params) + ">"]


def kernel_head(prog, name, temps, launch_bounds=DEFAULT_BLOCK, extra_params=()):
    params = kernel_params(prog, temps) + list(extra_params)
    return template_line(prog) + [
        f"__global__ void __launch_bounds__({launch_bounds}) {name}({', '.join(params)}) {{"
    ]


def arg_names(prog: lir.Program, temps):
    return [prog.output.name] + [n for n, _ in prog.inputs] + [t.name for t in temps]


# ---------------------------------------------------------------------------
# whole units


def _stage_buffers(stmt) -> set:
    out = set()
    for t, v in lir.stmt_exprs(stmt):
        if isinstance(t, lir.Store):
            out.add(t.buf)
        out.update(ld.buf for ld in lir.expr_loads(v))
    return out


def reuse_slots(stages, temps) -> dict:
    """Memory reuse of the Global temporaries (toMem(Global) between kernel
    stages): a temporary lives from the first to the last stage that touches
    it, and temporaries whose lives do not overlap share one allocation
    (greedy first fit in order of first use).  -> {temp name: slot index}."""
    life = {}
    for st in stages:
        for b in _stage_buffers(st.stmt):
            lo, hi = life.get(b, (st.index, st.index))
            life[b] = (min(lo, st.index), max(hi, st.index))
    slots = []  # per slot: the last stage index of its current occupant
    out = {}
    for t in sorted(temps, key=lambda t: life.get(t.name, (-1, -1))):
        lo, hi = life.get(t.name, (-1, -1))
        for k, end in enumerate(slots):
            if end < lo:
                slots[k] = hi
                out[t.name] = k
                break
        else:
            out[t.name] = len(slots)
            slots.append(hi)
    return out


class SingleBlockStage(UserWarning):
    """A kernel stage that runs in one block / one thread on the GPU."""


def emit_cuda(unit, exact=True, idioms=True, reassociate=True, peer_ranks=0, peer_halo=False,
              peer_out=0) -> CudaCode:
    """Emit the sm100a kernel text (and launch plan) for an ImperativeUnit.

    `reassociate=False` keeps every reduction in the program's own order
    (templates that reassociate — `reduce`, `gemm_tc`, fast-math `allpairs` —
    are not used), so every kernel is bit-exact with the reference's
    sequential semantics.

    `peer_ranks=R` (multi-GPU, one process per GPU): the `allpairs` source
    streams are distributed over R ranks in equal contiguous blocks and read
    in place through a device table of peer pointers (extra launch argument
    `rs_peer_table`), fusing the all-gather of the sources into the fold.

    `peer_out=R` (multi-GPU row bands whose result is all-gathered): the
    `rowfold` template also stores every row's value into every rank's
    full-result buffer (extra launch arguments `rs_y_table`: R peer pointers
    and this rank's row offset; `rs_peer_table`: the completion slots), and
    the ranks meet once per launch in epoch-tagged slots — the all-gather
    fused into the GEMV.

    `peer_halo=True` (multi-GPU row bands): the `stencil2d` template reads
    the rows padClamp would invent above / below the band from the
    neighbours' bands in place (extra launch arguments `rs_halo_top` /
    `rs_halo_bot`: peer pointers to their edge rows, or NULL at the image's
    real edges), fusing the halo exchange into the stencil."""
    from . import idioms as idiom_mod

    prog = lir.build(unit)
    prog.peer_ranks = int(peer_ranks)
    prog.peer_halo = bool(peer_halo)
    prog.peer_out = int(peer_out)
    prog.reassociate = bool(reassociate)  # (rowfold: split rows for short row counts)
    stages, temps = split_stages(prog.body, prog)
    kernels = []
    plan_stages = []
    includes = ["rise/device.cuh"]
    for st in stages:
        base = f"{prog.name}Kernel" if len(stages) == 1 else f"{prog.name}Kernel_s{st.index}"
        generic = GenericKernel(prog, st, base, temps, exact).emit()
        kernels.append(generic.text)
        entry = dict(generic.plan)
        match = idiom_mod.match(prog, st, base, temps, exact, reassociate) if idioms else None
        if peer_ranks and (match is None or not match.plan.get("peer_ranks")):
            raise EmitError("peer_ranks needs a stage the allpairs template (sources read in place) or the "
                            "reduce template (totals exchanged in peer memory) takes")
        if peer_halo and (match is None or not match.plan.get("peer_halo")):
            raise EmitError("peer_halo needs a stage the stencil2d template takes (halo rows read in place)")
        if peer_out and (match is None or not match.plan.get("peer_out")):
            raise EmitError("peer_out needs a stage the rowfold template takes (rows stored into every rank)")
        if match is not None:
            kernels.append(match.text)
            for inc in match.includes:
                if inc not in includes:
                    includes.append(inc)
            entry = dict(match.plan, fallback=generic.plan)
        else:
            # vector views (asVector / asScalar): the same kernel with float2 /
            # float4 accesses, the scalar kernel kept as its fallback
            vec = GenericKernel(prog, st, base + "_vec", temps, exact, vectorize=True)
            vtext = vec.emit()
            if vec.vector_accesses:
                kernels.append(vtext.text)
                entry = dict(vtext.plan, fallback=generic.plan, vector=True)
        if match is None and st.kind in ("block", "serial"):
            # a top-level sequential loop (or fold) no template claims runs in ONE
            # block (one thread for "serial"): correct, but a performance cliff
            entry["single_block"] = True
            warnings.warn(f"{base}: stage {st.index} runs as a single-{'block' if st.kind == 'block' else 'thread'} "
                          "kernel (a top-level sequential loop no template claims)", SingleBlockStage, stacklevel=2)
        plan_stages.append(entry)
    if PDL and len(stages) > 1:
        # programmatic dependent launch: stage k > 0 may be scheduled while
        # stage k - 1 drains; its first act is to wait for that grid's
        # completion and memory (a no-op when launched without the attribute)
        for k in range(1, len(plan_stages)):
            for st_plan in (plan_stages[k], plan_stages[k].get("fallback")):
                if st_plan:
                    st_plan["pdl"] = True
        def names(stage_plans):
            return [p["name"] for p in stage_plans] + [p["fallback"]["name"] for p in stage_plans if p.get("fallback")]
        # every stage but the last lets its dependent be scheduled at once: the
        # dependent's wait still covers this grid's completion and memory
        kernels = [_pdl_insert(kt, names(plan_stages[:-1]), "griddepcontrol.launch_dependents;",
                               "PDL: the next stage may be scheduled")
                   for kt in kernels]
        kernels = [_pdl_insert(kt, names(plan_stages[1:]), "griddepcontrol.wait;",
                               "PDL: the previous stage is done")
                   for kt in kernels]
    slot_of = reuse_slots(stages, temps)
    plan = {
        "version": 1,
        "target": TARGET,
        "unit": prog.name,
        "nat_params": list(prog.nat_params),
        "args": arg_names(prog, temps),
        "output": {"name": prog.output.name, "ctype": prog.output.ctype,
                   "size": py_expr(_prod(prog.output.dims)), "deref": prog.output.deref},
        "inputs": [_input_plan(n, b) for n, b in prog.inputs],
        "temps": [{"name": t.name, "ctype": t.ctype, "size": py_expr(_prod(t.dims)), "slot": slot_of[t.name]}
                  for t in temps],
        "stages": plan_stages,
        "exact": exact,
        "reassociate": reassociate,
    }
    if peer_halo:
        plan["peer_halo"] = True
    if peer_out:
        plan["peer_out"] = int(peer_out)
    if peer_ranks:
        plan["peer_ranks"] = int(peer_ranks)
        peers = {b for st in plan_stages for b in st.get("peer_streams", [])}
        for spec in plan["inputs"]:
            if spec["name"] in peers:
                spec["peer"] = True
    header = [
        f"// rise-b200 {TARGET} kernels for RISE unit '{prog.name}' (generated by emit_cuda; do not edit)",
        PLAN_TAG + json.dumps(plan, sort_keys=True),
    ] + [f"#include <{inc}>" for inc in includes]
    text = "\n".join(header) + "\n\n" + "\n".join(kernels)
    return CudaCode(text, plan, prog)


PDL = os.environ.get("RISE_PDL", "1") == "1"


def _pdl_insert(text, names, insn, why):
    """Insert the PTX `insn` as the first statement of the kernels named in
    `names` (their `__global__ ... name(...) {` line)."""
    out = []
    for line in text.split("\n"):
        out.append(line)
        if line.startswith("__global__") and line.rstrip().endswith("{") and \
                any(f" {n}(" in line for n in names):
            out.append(f'  asm volatile("{insn}" ::: "memory");  // {why}')
    return "\n".join(out)


def _prod(dims):
    out = nat.Const(1)
    for d in dims:
        out = out * d
    return nat.normalize(out)


def _input_plan(name, b):
    if isinstance(b, lir.ScalarRef):
        return {"name": name, "ctype": b.ctype, "scalar": True}
    return {"name": name, "ctype": b.ctype, "scalar": False, "size": py_expr(_prod(b.dims))}


def emit(unit, target: str = TARGET) -> str:
    """Drop-in for codegen.emit(unit, target) (codegen.py:451) with the new
    `sm100a` target.  (The reference target name "cuda" is not used: the
    reference suite asserts emit(unit, "cuda") raises, test_codegen.py:151.)"""
    if target != TARGET:
        from ._ref import codegen

        return codegen.emit(unit, target)
    return emit_cuda(unit).text


def plan_of(text: str) -> dict:
    for line in text.splitlines():
        if line.startswith(PLAN_TAG):
            return json.loads(line[len(PLAN_TAG):])
    raise errors.InterpreterError("kernel text carries no launch plan (not produced by emit_cuda)")
