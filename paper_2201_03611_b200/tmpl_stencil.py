"""`stencil2d` template: a 2-D parallel map whose body reads a 2-D array
through clamped neighbourhood indices (padClamp2D + slide2D programs).

Matches a stage whose parallel loops collapse to exactly two variables
(r < R, c < C) and in which every load of some 2-D array A has per-dimension
indices  clamp(r + o0, H-1)  and  clamp(c + o1, W-1),  where o0 / o1 are
affine in sequential loop variables with constant bounds (the window
offsets).  The offsets' ranges [omin, omax] give the halo.

Order: PRESERVED.  The body is the generic emitter's code for the program's
own loop nest (row sums, then the fold of the row sums, with the
round-to-nearest intrinsics); only the loads of A are redirected to a
shared-memory tile.  Bit-identical to the reference's semantics.

Data movement: one block computes a TR x TC output tile (32 x 8 threads,
RPT consecutive rows per thread so window rows are reused from registers);
the (TR + halo) x (TC + halo) input footprint is staged once into shared
memory, with the clamp applied while staging (padClamp semantics, so border
tiles need no special case).  Stores are 128-byte coalesced rows.
"""

from __future__ import annotations

from . import lir
from ._ref import nat
from .emit_cuda import GenericKernel, NatRenderer, Stage, ValueRenderer, kernel_head, py_expr

TC = 32  # columns per tile = blockDim.x
TY = 8  # blockDim.y
RPT = 8  # consecutive output rows per thread
TR = TY * RPT


def _seq_loop_bounds(stmt):
    out = {}
    for s in lir.walk(stmt):
        if isinstance(s, (lir.For, lir.ParFor)):
            out[s.var] = s.bound
    return out


def _offset_range(expr, base_var, loop_bounds):
    """expr = base_var + off with off affine in loop vars of constant bound:
    (omin, omax) or None."""
    if base_var not in nat.free_vars(expr):
        return None
    off = nat.normalize(expr - nat.Var(base_var))
    if base_var in nat.free_vars(off):
        return None
    lo = hi = nat.normalize(nat.substitute(off, {v: nat.Const(0) for v in nat.free_vars(off)}))
    if not isinstance(lo, nat.Const):
        return None
    lo = hi = lo.value
    for v in nat.free_vars(off):
        b = loop_bounds.get(v)
        if b is None or not isinstance(b, nat.Const) or b.value < 1:
            return None
        zero = {u: nat.Const(0) for u in nat.free_vars(off)}
        one = dict(zero)
        one[v] = nat.Const(1)
        coef = nat.normalize(nat.substitute(off, one) - nat.substitute(off, zero))
        two = dict(zero)
        two[v] = nat.Const(2)
        coef2 = nat.normalize(nat.substitute(off, two) - nat.substitute(off, zero))
        if not (isinstance(coef, nat.Const) and isinstance(coef2, nat.Const) and coef2.value == 2 * coef.value):
            return None
        span = coef.value * (b.value - 1)
        lo += min(0, span)
        hi += max(0, span)
    return lo, hi


def match(prog, stage, base_name, temps, exact, parallel_rows):
    loops, body = parallel_rows(stage)
    if loops is None or len(loops) != 2 or stage.kind != "grid":
        return None
    (rv, R), (cv, C) = loops
    bounds = _seq_loop_bounds(body)
    tiled = {}  # buf -> [omin0, omax0, omin1, omax1, H-1, W-1]
    for _t, value in lir.stmt_exprs(body):
        for ld in lir.expr_loads(value):
            if not any(v in prog.clamps for v in nat.free_vars(ld.index)):
                if rv in nat.free_vars(ld.index) or cv in nat.free_vars(ld.index):
                    if ld.buf in tiled:
                        return None
                continue
            buf = prog.buffers[ld.buf]
            if buf.role != "input" or len(buf.dims) != 2 or len(ld.indices) != 2:
                return None
            e0, e1 = ld.indices
            if not (isinstance(e0, nat.Var) and e0.name in prog.clamps and isinstance(e1, nat.Var)
                    and e1.name in prog.clamps):
                return None
            (in0, hi0), (in1, hi1) = prog.clamps[e0.name], prog.clamps[e1.name]
            if not (nat.equal(hi0, nat.normalize(buf.dims[0] - nat.Const(1)))
                    and nat.equal(hi1, nat.normalize(buf.dims[1] - nat.Const(1)))):
                return None
            r0 = _offset_range(in0, rv, bounds)
            r1 = _offset_range(in1, cv, bounds)
            if r0 is None or r1 is None:
                return None
            cur = tiled.setdefault(ld.buf, [r0[0], r0[1], r1[0], r1[1]])
            cur[0], cur[1] = min(cur[0], r0[0]), max(cur[1], r0[1])
            cur[2], cur[3] = min(cur[2], r1[0]), max(cur[3], r1[1])
    if len(tiled) != 1:
        return None
    (abuf, (o0lo, o0hi, o1lo, o1hi)), = tiled.items()
    if o0hi - o0lo > 16 or o1hi - o1lo > 16:
        return None
    A = prog.buffers[abuf]
    name = f"{base_name}_stencil"
    r = NatRenderer(prog.clamps)
    HR = TR + (o0hi - o0lo)
    HC = TC + (o1hi - o1lo)

    def hook(ld):
        if ld.buf != abuf:
            return None
        e0, e1 = ld.indices
        in0 = prog.clamps[e0.name][0]
        in1 = prog.clamps[e1.name][0]
        return f"rs_tile[(({r(in0)}) - rs_tr0) * {HC} + (({r(in1)}) - rs_tc0)]"

    g = GenericKernel(prog, Stage("serial", body), "_", [], exact)
    g.r = ValueRenderer(prog, exact, load_hook=hook)
    body_lines = g.thread(body, 3)

    lines = kernel_head(prog, name, temps, launch_bounds=TC * TY)
    lines += [
        f"  constexpr int RS_R = {r(R)}, RS_C = {r(C)};",
        f"  __shared__ float rs_tile[{HR} * {HC}];",
        f"  const int rs_r0 = blockIdx.y * {TR}, rs_c0 = blockIdx.x * {TC};",
        f"  const int rs_tr0 = rs_r0 + ({o0lo}), rs_tc0 = rs_c0 + ({o1lo});",
        f"  for (int rs_e = threadIdx.y * {TC} + threadIdx.x; rs_e < {HR * HC}; rs_e += {TC * TY}) {{",
        f"    const int rs_y = rs_e / {HC}, rs_x = rs_e % {HC};",
        f"    rs_tile[rs_e] = {abuf}[rs_clamp(rs_tr0 + rs_y, {r(nat.normalize(A.dims[0] - nat.Const(1)))}) * "
        f"({r(A.dims[1])}) + rs_clamp(rs_tc0 + rs_x, {r(nat.normalize(A.dims[1] - nat.Const(1)))})];",
        "  }",
        "  __syncthreads();",
        f"  const int {cv} = rs_c0 + threadIdx.x;",
        f"  if (rs_r0 + {TR} <= RS_R && rs_c0 + {TC} <= RS_C) {{",
        "    // interior tile: unguarded, so window loads are shared across the unrolled rows",
        "#pragma unroll",
        f"    for (int rs_k = 0; rs_k < {RPT}; ++rs_k) {{",
        f"      const int {rv} = rs_r0 + threadIdx.y * {RPT} + rs_k;",
        "      {",
    ]
    lines += ["    " + x for x in body_lines]
    lines += [
        "      }",
        "    }",
        "  } else {",
        f"    for (int rs_k = 0; rs_k < {RPT}; ++rs_k) {{",
        f"      const int {rv} = rs_r0 + threadIdx.y * {RPT} + rs_k;",
        f"      if ({rv} < RS_R && {cv} < RS_C) {{",
    ]
    lines += ["    " + x for x in body_lines]
    lines += ["      }", "    }", "  }", "}"]
    plan = {
        "name": name,
        "kind": "stencil2d",
        "rows": py_expr(R),
        "cols": py_expr(C),
        "tile": [TR, TC],
        "block": [TC, TY],
        "fmad": False,
        "order": "preserved",
        "pre": [],
    }
    return "\n".join(lines) + "\n", plan


def launch(st, nats, sm):
    from .emit_cuda import eval_py

    rows = eval_py(st["rows"], nats)
    cols = eval_py(st["cols"], nats)
    tr, tc = st["tile"]
    return (-(-cols // tc), -(-rows // tr), 1), (st["block"][0], st["block"][1], 1), 0, (1, 1, 1)
