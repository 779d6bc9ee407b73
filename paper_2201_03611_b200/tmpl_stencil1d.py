"""`stencil1d` template: a 1-D parallel map whose body reads a 1-D input
through clamped window indices (padClamp + slide programs: `slide1D`, 1-D
smoothing, finite differences).

Matches a stage with ONE parallel loop (i < N) in which every load of some
1-D float input A has the index  clamp(i + o, H - 1)  with o affine in
sequential loop variables of constant bound (the window), and no other load
depends on i.  The generic kernel reads each window element from global
memory through the clamp (three loads per output for a 3-window, two of
them misaligned): ≈ 3.7 TB/s at 2^26 (`tools/probe_transpose.py`).

Data movement: a block owns TN = 4096 consecutive outputs.  One elected
thread stages the footprint A[i0 - LP, i0 + TN + RP) (LP / RP: the window's
reach, rounded up to 16 bytes) into shared memory with ONE 1-D bulk copy of
its in-range part; at the array's ends the block applies padClamp in shared
memory (cells before 0 take A[0], cells past H - 1 take A[H - 1]).  Thread t
then computes outputs t, t + 256, ... of the tile with the program's own
body, its loads of A redirected to the staged cells (conflict-free LDS),
and stores them coalesced.

Order: PRESERVED — the body is the program's own, on the same values.
Bit-identical to the reference's semantics.
"""

from __future__ import annotations

from . import lir
from ._ref import nat
from .emit_cuda import GenericKernel, NatRenderer, Stage, ValueRenderer, kernel_head, py_expr
from .tmpl_stencil import _offset_range, _seq_loop_bounds

TN = 4096  # outputs per block
BLOCK = 256


def match(prog, stage, base_name, temps, exact, parallel_rows):
    if stage.kind != "grid":
        return None
    loops, body = parallel_rows(stage)
    if loops is None or len(loops) != 1:
        return None
    ((iv, N),) = loops
    bounds = _seq_loop_bounds(body)
    abuf, lo, hi = None, None, None
    unclamped = set()  # buffers also read at indices that are not clamp variables
    for _t, value in lir.stmt_exprs(body):
        for ld in lir.expr_loads(value):
            clamped = [v for v in nat.free_vars(ld.index) if v in prog.clamps]
            if not clamped:
                if iv in nat.free_vars(ld.index):
                    return None  # another i-dependent stream: the generic kernel keeps it
                unclamped.add(ld.buf)
                continue
            buf = prog.buffers[ld.buf]
            if buf.role != "input" or buf.ctype != "float" or len(buf.dims) != 1 or len(ld.indices) != 1:
                return None
            e0 = ld.indices[0]
            if not (isinstance(e0, nat.Var) and e0.name in prog.clamps):
                return None
            inner, top = prog.clamps[e0.name]
            if not nat.equal(top, nat.normalize(buf.dims[0] - nat.Const(1))):
                return None
            rng = _offset_range(inner, iv, bounds)
            if rng is None or (abuf is not None and abuf != ld.buf):
                return None
            abuf = ld.buf
            lo = rng[0] if lo is None else min(lo, rng[0])
            hi = rng[1] if hi is None else max(hi, rng[1])
    if abuf is None or not (lo <= 0 <= hi) or hi - lo > 64:
        return None
    if abuf in unclamped:
        return None  # e.g. A[0] or A[k] beside the window: only clamped loads are redirected to the tile
    A = prog.buffers[abuf]
    H = A.dims[0]
    r = NatRenderer(prog.clamps)
    lp = -(-(-lo) // 4) * 4  # staged cells before the tile (16-byte multiple)
    rp = -(-hi // 4) * 4
    sl = TN + lp + rp

    def hook(ld):
        if ld.buf != abuf:
            return None
        off = nat.normalize(prog.clamps[ld.indices[0].name][0] - nat.Var(iv))
        return f"rs_tile[rs_li + ({r(off)}) + {lp}]"

    g = GenericKernel(prog, Stage("serial", body), "_", [], exact)
    g.r = ValueRenderer(prog, exact, load_hook=hook)
    body_lines = g.thread(body, 3)
    name = f"{base_name}_stencil1d"
    lines = kernel_head(prog, name, temps, launch_bounds=BLOCK)
    lines += [
        f"  constexpr int RS_N = {r(N)}, RS_H = {r(H)}, RS_TN = {TN}, RS_LP = {lp}, RS_SL = {sl};",
        "  __shared__ __align__(128) float rs_tile[RS_SL];",
        "  __shared__ __align__(8) unsigned long long rs_bar;",
        "  const int rs_i0 = blockIdx.x * RS_TN, rs_s0 = rs_i0 - RS_LP;  // staged cell k holds A[rs_s0 + k]",
        "  const int rs_cs = rs_s0 < 0 ? 0 : rs_s0, rs_ce = rs_s0 + RS_SL > RS_H ? RS_H : rs_s0 + RS_SL;",
        "  if (threadIdx.x == 0) {",
        "    rs_mbar_init(&rs_bar, 1);",
        "    rs_fence_barrier_init();",
        "    rs_mbar_arrive_expect_tx(&rs_bar, (unsigned)((rs_ce - rs_cs) * 4));",
        f"    rs_bulk_g2s(rs_tile + (rs_cs - rs_s0), {abuf} + rs_cs, (unsigned)((rs_ce - rs_cs) * 4), &rs_bar);",
        "  }",
        "  __syncthreads();",
        "  rs_mbar_wait(&rs_bar, 0);",
        "  if (rs_s0 < 0 || rs_s0 + RS_SL > RS_H) {  // padClamp at the array's ends",
        f"    for (int rs_k = threadIdx.x; rs_k < RS_SL; rs_k += {BLOCK}) {{",
        "      const int rs_g = rs_s0 + rs_k;",
        "      if (rs_g < 0) rs_tile[rs_k] = rs_tile[-rs_s0];",
        "      else if (rs_g >= RS_H) rs_tile[rs_k] = rs_tile[RS_H - 1 - rs_s0];",
        "    }",
        "    __syncthreads();",
        "  }",
        "#pragma unroll 4",
        f"  for (int rs_q = 0; rs_q < RS_TN / {BLOCK}; ++rs_q) {{",
        f"    const int rs_li = rs_q * {BLOCK} + threadIdx.x;",
        f"    const int {iv} = rs_i0 + rs_li;",
        f"    if ({iv} < RS_N) {{",
    ]
    lines += body_lines
    lines += ["    }", "  }", "}"]
    pre = [f"({py_expr(H)}) % 4 == 0", f"({py_expr(N)}) <= ({py_expr(H)})", f"({py_expr(N)}) > 0"]
    plan = {
        "name": name,
        "kind": "stencil1d",
        "rows": py_expr(N),
        "block": BLOCK,
        "fmad": False,
        "order": "preserved",
        "pre": pre,
    }
    return "\n".join(lines) + "\n", plan


def launch(st, nats, sm):
    from .emit_cuda import eval_py

    n = eval_py(st["rows"], nats)
    return (max(1, -(-n // TN)), 1, 1), (st["block"], 1, 1), 0, (1, 1, 1)
