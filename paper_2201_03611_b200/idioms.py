"""Idiom matching: LIR stages -> hand-written sm_100a kernel templates.

A template is chosen only when the stage's loop nest has exactly the shape
the template implements; otherwise the generic kernel (emit_cuda.py) runs.
Each template keeps or states the program's evaluation order:

* `rowfold` — a parallel map over rows whose body is a sequential fold
  `acc = step(acc, loads(row, j))` over j < K, with every j-dependent load
  unit-stride in j (gemv `mv.rise`, the paper's `mv_opt` schedule, chunked
  reductions).  The fold order is PRESERVED: one thread folds one row, in
  j order, with the program's own step expression; what the template adds
  is the data movement — row segments and row-invariant segments are
  streamed through a multi-stage shared-memory ring by the TMA bulk-copy
  engine (cp.async.bulk + mbarrier), so the per-thread sequential loop reads
  conflict-free shared memory instead of stride-K global memory.  Results
  are bit-identical to the reference's sequential semantics.
* `reduce` — a top-level sequential fold `acc = acc + term(i)` over the
  whole input (the `dot` program after `toReduceSeq`).  One sequential chain
  of 2^24 dependent adds cannot run in parallel in its own order, so this
  template REASSOCIATES `+` into a fixed, documented tree (DESIGN.md
  "Reduction order"): per-thread left folds over a fixed strided float4
  partition, a warp butterfly, a block butterfly, and a last-block fold of
  the block partials.  The order depends only on the problem size, never on
  scheduling; parity is the fp64 error bound of SURVEY.md §8 d.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from . import lir
from ._ref import nat
from .emit_cuda import (
    NatRenderer,
    ValueRenderer,
    collapse_global_chain,
    kernel_head,
    py_expr,
)


@dataclass
class IdiomKernel:
    name: str
    text: str
    plan: dict
    includes: list = field(default_factory=list)


def match(prog, stage, base_name, temps, exact):
    for matcher in (_match_rowfold, _match_reduce):
        out = matcher(prog, stage, base_name, temps, exact)
        if out is not None:
            return out
    return None


# ---------------------------------------------------------------------------
# shared analysis helpers


def _parallel_rows(stage):
    """Collapse the stage's parallel loops into rows: ([(var, bound)], body)."""
    s = stage.stmt
    if stage.kind == "grid":
        return collapse_global_chain(s)
    if stage.kind == "workgroup":
        loops = [(s.var, s.bound)]
        body = s.body
        if isinstance(body, lir.ParFor) and body.kind == "local":
            loops.append((body.var, body.bound))
            return loops, body.body
    return None, None


def _fold_shape(body):
    """Alloc(acc scalar) { acc = INIT; for j < K: acc = STEP; POST... }"""
    if not (isinstance(body, lir.Alloc) and body.dims == () and body.space == "Private"):
        return None
    acc = lir.ScalarRef(body.name, body.ctype)
    stmts = body.body.stmts if isinstance(body.body, lir.Seq) else [body.body]
    if len(stmts) < 2:
        return None
    init, loop, post = stmts[0], stmts[1], stmts[2:]
    if not (isinstance(init, lir.Assign) and init.target == acc):
        return None
    if acc in set(lir.expr_scalars(init.value)):
        return None
    if not (isinstance(loop, lir.For) and isinstance(loop.body, lir.Assign) and loop.body.target == acc):
        return None
    for s in post:
        for t in lir.walk(s):
            if isinstance(t, (lir.For, lir.ParFor, lir.DoubleBuffer, lir.Alloc)):
                return None
    return acc, init, loop, post


def _j_coefficient(index, j):
    """0 if `index` does not use j, 1 if index == base + j, else None."""
    jv = nat.Var(j)
    if j not in nat.free_vars(index):
        return 0, index
    base = nat.normalize(nat.substitute(index, {j: nat.Const(0)}))
    if nat.equal(nat.normalize(base + jv), nat.normalize(index)) and j not in nat.free_vars(base):
        return 1, base
    return None, None


def _uses_clamp(n, prog):
    return any(v in prog.clamps for v in nat.free_vars(n))


def _coeff_preconditions(base, row_vars, align=4):
    """Python preconditions: base(row) % align == 0 for every row, assuming
    base is affine in the row variables (checked by second differences)."""
    zero = {v: nat.Const(0) for v in row_vars}
    c0 = nat.normalize(nat.substitute(base, zero))
    pre = [f"({py_expr(c0)}) % {align} == 0"]
    for v in row_vars:
        one = dict(zero)
        one[v] = nat.Const(1)
        two = dict(zero)
        two[v] = nat.Const(2)
        c1 = nat.normalize(nat.substitute(base, one) - c0)
        c2 = nat.normalize(nat.substitute(base, two) - c0)
        if not nat.equal(c2, nat.normalize(c1 * nat.Const(2))):
            return None  # not affine in v
        pre.append(f"({py_expr(c1)}) % {align} == 0")
    return pre


def _row_decomp(loops, flat="rs_f"):
    """Lines decomposing a flat row index into the collapsed loop variables."""
    r = NatRenderer()
    lines = []
    rest = flat
    for k, (var, _bound) in enumerate(loops):
        if k == len(loops) - 1:
            lines.append(f"const int {var} = {rest};")
        else:
            inner = nat.Const(1)
            for _, b in loops[k + 1:]:
                inner = inner * b
            size_c = r(nat.normalize(inner), 2)
            lines.append(f"const int {var} = {rest} / {size_c};")
            lines.append(f"const int rs_q{k} = {rest} % {size_c};")
            rest = f"rs_q{k}"
    return lines


# ---------------------------------------------------------------------------
# rowfold


ROWFOLD_ROWS = 32
ROWFOLD_KT = 128
ROWFOLD_STAGES = 4


def _match_rowfold(prog, stage, base_name, temps, exact):
    loops, body = _parallel_rows(stage)
    if loops is None:
        return None
    shape = _fold_shape(body)
    if shape is None:
        return None
    acc, init, loop, post = shape
    j = loop.var
    row_vars = [v for v, _ in loops]
    step = loop.body.value
    loads = list(dict.fromkeys(lir.expr_loads(step)))
    row_streams = {}  # Load -> (buf, base)
    shared_streams = {}
    for ld in loads:
        if _uses_clamp(ld.index, prog):
            return None
        coef, base = _j_coefficient(ld.index, j)
        if coef is None:
            return None
        if coef == 0:
            continue  # j-invariant: read directly
        buf = prog.buffers[ld.buf]
        if buf.role == "pointer" or (buf.role == "alloc" and buf.space != "Global"):
            return None
        if any(v in nat.free_vars(base) for v in row_vars):
            row_streams[ld] = (ld.buf, base)
        else:
            if any(v in nat.free_vars(base) for v in [j]):
                return None
            shared_streams[ld] = (ld.buf, base)
    if not row_streams:
        return None
    # every streamed load must only depend on row variables and sizes
    allowed = set(row_vars) | set(prog.nat_params)
    for ld, (_b, base) in list(row_streams.items()) + list(shared_streams.items()):
        if not nat.free_vars(base) <= allowed:
            return None
    pre = [f"({py_expr(loop.bound)}) % 4 == 0"]
    for ld, (_b, base) in list(row_streams.items()) + list(shared_streams.items()):
        p = _coeff_preconditions(base, row_vars if ld in row_streams else [])
        if p is None:
            return None
        pre += p
    pre = list(dict.fromkeys(pre))

    name = f"{base_name}_rowfold"
    r = NatRenderer(prog.clamps)
    nrows = nat.Const(1)
    for _, b in loops:
        nrows = nrows * b
    nrows = nat.normalize(nrows, prog.assumptions)

    rs_list = list(dict.fromkeys((b, base) for b, base in row_streams.values()))
    sh_list = list(dict.fromkeys((b, base) for b, base in shared_streams.values()))
    R, KT, S = ROWFOLD_ROWS, ROWFOLD_KT, ROWFOLD_STAGES
    LD = KT + 4

    lines = kernel_head(prog, name, temps, launch_bounds=R)
    lines += [
        f"  constexpr int RS_ROWS = {R}, RS_KT = {KT}, RS_STAGES = {S}, RS_LD = {LD};",
        f"  constexpr int RS_NROWS = {r(nrows)};",
        f"  constexpr int RS_K = {r(loop.bound)};",
        "  constexpr int RS_NT = (RS_K + RS_KT - 1) / RS_KT;",
        "  extern __shared__ __align__(128) unsigned char rs_smem[];",
    ]
    off = "0"
    for k in range(len(rs_list)):
        lines.append(f"  float* rs_sa{k} = reinterpret_cast<float*>(rs_smem) + {off};")
        off = f"{off} + RS_STAGES * RS_ROWS * RS_LD"
    for k in range(len(sh_list)):
        lines.append(f"  float* rs_sx{k} = reinterpret_cast<float*>(rs_smem) + {off};")
        off = f"{off} + RS_STAGES * RS_KT"
    lines += [
        f"  unsigned long long* rs_bar = reinterpret_cast<unsigned long long*>(reinterpret_cast<float*>(rs_smem) + {off});",
        "  const int rs_lane = threadIdx.x;",
        "  const int rs_row0 = blockIdx.x * RS_ROWS;",
        "  const bool rs_active = rs_row0 + rs_lane < RS_NROWS;",
        "  const int rs_nact = RS_NROWS - rs_row0 < RS_ROWS ? RS_NROWS - rs_row0 : RS_ROWS;",
        "  const int rs_f = rs_active ? rs_row0 + rs_lane : RS_NROWS - 1;",
    ]
    lines += ["  " + x for x in _row_decomp(loops)]
    for k, (buf, base) in enumerate(rs_list):
        lines.append(f"  const float* rs_ga{k} = {buf} + ({r(base)});")
    for k, (buf, base) in enumerate(sh_list):
        lines.append(f"  const float* rs_gx{k} = {buf} + ({r(base)});")
    nstream = len(sh_list)
    lines += [
        "  if (rs_lane == 0) {",
        "    for (int rs_s = 0; rs_s < RS_STAGES; ++rs_s) rs_mbar_init(&rs_bar[rs_s], 1);",
        "    rs_fence_barrier_init();",
        "  }",
        "  __syncwarp();",
        "  auto rs_issue = [&](int rs_t) {",
        "    const int rs_slot = rs_t % RS_STAGES;",
        "    const int rs_j0 = rs_t * RS_KT;",
        "    const int rs_kt = RS_K - rs_j0 < RS_KT ? RS_K - rs_j0 : RS_KT;",
        "    const unsigned rs_bytes = (unsigned)rs_kt * 4u;",
        "    rs_fence_proxy_async();",
        f"    if (rs_lane == 0) rs_mbar_arrive_expect_tx(&rs_bar[rs_slot], rs_bytes * (unsigned)(rs_nact * {len(rs_list)} + {nstream}));",
        "    __syncwarp();",
        "    if (rs_active) {",
    ]
    for k in range(len(rs_list)):
        lines.append(f"      rs_bulk_g2s(rs_sa{k} + (rs_slot * RS_ROWS + rs_lane) * RS_LD, rs_ga{k} + rs_j0, rs_bytes, &rs_bar[rs_slot]);")
    lines.append("    }")
    if sh_list:
        lines.append("    if (rs_lane == 0) {")
        for k in range(len(sh_list)):
            lines.append(f"      rs_bulk_g2s(rs_sx{k} + rs_slot * RS_KT, rs_gx{k} + rs_j0, rs_bytes, &rs_bar[rs_slot]);")
        lines.append("    }")
    lines += [
        "  };",
        "  for (int rs_t = 0; rs_t < RS_STAGES - 1 && rs_t < RS_NT; ++rs_t) rs_issue(rs_t);",
    ]
    vr = ValueRenderer(prog, exact)
    lines.append(f"  {acc.ctype} {acc.name};")
    lines.append(f"  {acc.name} = {vr(init.value)};")

    def step_with(comp):
        def hook(ld):
            if ld in row_streams:
                k = rs_list.index(row_streams[ld])
                return f"rs_a{k}.{comp}"
            if ld in shared_streams:
                k = sh_list.index(shared_streams[ld])
                return f"rs_x{k}.{comp}"
            return None

        return ValueRenderer(prog, exact, load_hook=hook)(step)

    def chunk(ind):
        p = " " * ind
        out = []
        for k in range(len(rs_list)):
            out.append(f"{p}const float4 rs_a{k} = *reinterpret_cast<const float4*>(rs_pa{k} + rs_jj);")
        for k in range(len(sh_list)):
            out.append(f"{p}const float4 rs_x{k} = *reinterpret_cast<const float4*>(rs_px{k} + rs_jj);")
        for comp in ("x", "y", "z", "w"):
            out.append(f"{p}{acc.name} = {step_with(comp)};")
        return out

    lines += [
        "  for (int rs_t = 0; rs_t < RS_NT; ++rs_t) {",
        "    if (rs_t + RS_STAGES - 1 < RS_NT) rs_issue(rs_t + RS_STAGES - 1);",
        "    const int rs_slot = rs_t % RS_STAGES;",
        "    rs_mbar_wait(&rs_bar[rs_slot], (unsigned)((rs_t / RS_STAGES) & 1));",
    ]
    for k in range(len(rs_list)):
        lines.append(f"    const float* rs_pa{k} = rs_sa{k} + (rs_slot * RS_ROWS + rs_lane) * RS_LD;")
    for k in range(len(sh_list)):
        lines.append(f"    const float* rs_px{k} = rs_sx{k} + rs_slot * RS_KT;")
    lines += [
        "    const int rs_kt = RS_K - rs_t * RS_KT < RS_KT ? RS_K - rs_t * RS_KT : RS_KT;",
        "    if (rs_kt == RS_KT) {",
        "#pragma unroll 8",
        "      for (int rs_jj = 0; rs_jj < RS_KT; rs_jj += 4) {",
    ]
    lines += chunk(8)
    lines += [
        "      }",
        "    } else {",
        "      for (int rs_jj = 0; rs_jj < rs_kt; rs_jj += 4) {",
    ]
    lines += chunk(8)
    lines += [
        "      }",
        "    }",
        "    __syncwarp();",
        "  }",
        "  if (rs_active) {",
    ]
    for s in post:
        lines += [("    " + x) for x in _thread_lines(prog, s, exact)]
    lines += ["  }", "}"]
    smem = (len(rs_list) * S * R * LD + len(sh_list) * S * KT) * 4 + S * 8
    plan = {
        "name": name,
        "kind": "rowfold",
        "rows": py_expr(nrows),
        "row_block": R,
        "smem": smem,
        "pre": pre,
        "fmad": False,
        "order": "preserved",
    }
    return IdiomKernel(name, "\n".join(lines) + "\n", plan)


def _thread_lines(prog, stmt, exact):
    from .emit_cuda import GenericKernel, Stage

    return GenericKernel(prog, Stage("serial", stmt), "_", [], exact).thread(stmt, 0)


def _launch_rowfold(st, nats, sm):
    from .emit_cuda import eval_py

    rows = eval_py(st["rows"], nats)
    grid = max(1, -(-rows // st["row_block"]))
    return (grid, 1, 1), (st["row_block"], 1, 1), st["smem"], (1, 1, 1)


# ---------------------------------------------------------------------------
# reduce (reassociated, deterministic)

REDUCE_GRID = 1184  # 8 x 148; fixed so the reduction order never depends on the GPU
REDUCE_BLOCK = 256


def _match_reduce(prog, stage, base_name, temps, exact):
    if stage.kind != "serial":
        return None
    shape = _fold_shape(stage.stmt)
    if shape is None:
        return None
    acc, init, loop, post = shape
    step = loop.body.value
    if not (isinstance(step, lir.Bin) and step.op == "+" and step.a == acc):
        return None
    term = step.b
    if acc in set(lir.expr_scalars(term)):
        return None
    i = loop.var
    loads = list(dict.fromkeys(lir.expr_loads(term)))
    streams = {}
    for ld in loads:
        if _uses_clamp(ld.index, prog):
            return None
        coef, base = _j_coefficient(ld.index, i)
        if coef is None:
            return None
        if coef == 1:
            if not nat.free_vars(base) <= set(prog.nat_params):
                return None
            streams[ld] = (ld.buf, base)
        elif not nat.free_vars(ld.index) <= set(prog.nat_params):
            return None
    if not streams:
        return None
    for s in post:  # post may only read the accumulator and write memory
        for t in lir.walk(s):
            if isinstance(t, lir.Assign) and isinstance(t.target, lir.ScalarRef) and t.target != acc:
                return None
    pre = [f"({py_expr(loop.bound)}) % 4 == 0"]
    for ld, (_b, base) in streams.items():
        pre.append(f"({py_expr(base)}) % 4 == 0")
    pre = list(dict.fromkeys(pre))
    s_list = list(dict.fromkeys(streams.values()))
    name = f"{base_name}_reduce"
    r = NatRenderer(prog.clamps)
    ct = acc.ctype
    zero = "0.0f" if ct == "float" else "0"
    vr_plain = ValueRenderer(prog, exact)

    def add(a, b):
        return f"__fadd_rn({a}, {b})" if (ct == "float" and exact) else f"({a} + {b})"

    def term_with(comp):
        def hook(ld):
            if ld in streams:
                return f"rs_v{s_list.index(streams[ld])}.{comp}"
            return None

        return ValueRenderer(prog, exact, load_hook=hook)(term)

    shfl = "__shfl_xor_sync(0xffffffffu, rs_s, rs_o)"
    lines = kernel_head(prog, name, temps, launch_bounds=REDUCE_BLOCK,
                        extra_params=[f"{ct}* __restrict__ rs_partials", "unsigned* __restrict__ rs_ticket"])
    lines += [
        f"  constexpr int RS_N4 = ({r(loop.bound)}) / 4;",
        f"  constexpr int RS_T = {REDUCE_GRID} * {REDUCE_BLOCK};",
        "  const int rs_tid = blockIdx.x * blockDim.x + threadIdx.x;",
    ]
    for k, (buf, base) in enumerate(s_list):
        lines.append(f"  const float4* __restrict__ rs_g{k} = reinterpret_cast<const float4*>({buf} + ({r(base)}));")
    lines += [
        f"  {ct} rs_acc = {zero};",
        "  // phase 1: thread-local left fold over float4 chunks tid, tid+T, tid+2T, ...",
        "#pragma unroll 4",
        "  for (int rs_c = rs_tid; rs_c < RS_N4; rs_c += RS_T) {",
    ]
    for k in range(len(s_list)):
        lines.append(f"    const float4 rs_v{k} = rs_ldg_stream(rs_g{k} + rs_c);")
    for comp in ("x", "y", "z", "w"):
        lines.append(f"    rs_acc = {add('rs_acc', term_with(comp))};")
    lines += [
        "  }",
        "  // phase 2: warp butterfly (xor 16, 8, 4, 2, 1); every lane ends with the same value",
        f"  {ct} rs_s = rs_acc;",
        "#pragma unroll",
        f"  for (int rs_o = 16; rs_o > 0; rs_o >>= 1) rs_s = {add('rs_s', shfl)};",
        f"  __shared__ {ct} rs_w[{REDUCE_BLOCK // 32}];",
        "  __shared__ bool rs_last;",
        "  if ((threadIdx.x & 31) == 0) rs_w[threadIdx.x >> 5] = rs_s;",
        "  __syncthreads();",
        "  // phase 3: block butterfly over the warp totals (warp 0)",
        "  if (threadIdx.x < 32) {",
        f"    rs_s = threadIdx.x < {REDUCE_BLOCK // 32} ? rs_w[threadIdx.x] : {zero};",
        "#pragma unroll",
        f"    for (int rs_o = 16; rs_o > 0; rs_o >>= 1) rs_s = {add('rs_s', shfl)};",
        "    if (threadIdx.x == 0) {",
        "      rs_partials[blockIdx.x] = rs_s;",
        "      __threadfence();",
        "      rs_last = atomicAdd(rs_ticket, 1u) == gridDim.x - 1;",
        "    }",
        "  }",
        "  __syncthreads();",
        "  if (!rs_last) return;",
        "  // phase 4 (last block): lane-strided left folds of the block partials, then butterflies",
        "  __threadfence();",
        f"  {ct} rs_p = {zero};",
        "  for (int rs_b = threadIdx.x; rs_b < gridDim.x; rs_b += blockDim.x) {",
        f"    rs_p = {add('rs_p', '__ldcg(rs_partials + rs_b)')};",
        "  }",
        "  rs_s = rs_p;",
        "#pragma unroll",
        f"  for (int rs_o = 16; rs_o > 0; rs_o >>= 1) rs_s = {add('rs_s', shfl)};",
        "  if ((threadIdx.x & 31) == 0) rs_w[threadIdx.x >> 5] = rs_s;",
        "  __syncthreads();",
        "  if (threadIdx.x < 32) {",
        f"    rs_s = threadIdx.x < {REDUCE_BLOCK // 32} ? rs_w[threadIdx.x] : {zero};",
        "#pragma unroll",
        f"    for (int rs_o = 16; rs_o > 0; rs_o >>= 1) rs_s = {add('rs_s', shfl)};",
        "    if (threadIdx.x == 0) {",
        f"      {ct} {acc.name} = {vr_plain(init.value)};",
        f"      {acc.name} = {add(acc.name, 'rs_s')};",
    ]
    for s in post:
        lines += [("      " + x) for x in _thread_lines(prog, s, exact)]
    lines += [
        "      *rs_ticket = 0u;",
        "    }",
        "  }",
        "}",
    ]
    ws_p = f"rs_ws_{base_name}_partials"
    ws_t = f"rs_ws_{base_name}_ticket"
    plan = {
        "name": name,
        "kind": "reduce",
        "grid": REDUCE_GRID,
        "block": REDUCE_BLOCK,
        "pre": pre,
        "fmad": False,
        "order": "reassociated",
        "workspace": [{"name": ws_p, "ctype": ct, "size": str(REDUCE_GRID)},
                      {"name": ws_t, "ctype": "int", "size": "1"}],
        "extra_args": [{"kind": "workspace", "name": ws_p}, {"kind": "workspace", "name": ws_t}],
    }
    return IdiomKernel(name, "\n".join(lines) + "\n", plan)


def _launch_reduce(st, nats, sm):
    return (st["grid"], 1, 1), (st["block"], 1, 1), 0, (1, 1, 1)


LAUNCHERS = {
    "rowfold": _launch_rowfold,
    "reduce": _launch_reduce,
}
