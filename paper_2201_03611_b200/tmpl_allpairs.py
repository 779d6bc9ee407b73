"""`allpairs` template: every target folds over every source (nbody).

Matches a grid stage over targets g < NT whose body is

    [for c < C:]                       # a small, constant component loop
      acc = INIT(g, c)
      for j < NS:  S(g, c, j, acc)      # any private computation ending in
                                        #   acc = f(acc, ...)
      POST(g, c, acc)                   # e.g. output[3g + c] = vel + dt * acc

where every load that depends on j reads a "source stream" B[a*j + off]
with a constant stride a and 0 <= off < a (off from c and constant inner
loops), and every other load is j-invariant (the target's own data).

Order: when the fold step is `acc = acc + e(j)`, the sources are split into
SPLIT contiguous chunks of ceil(NS/SPLIT): warp w of a block folds chunk w
in j order (chunk 0 from INIT, the others from +0.0) and the partials are
added in chunk order, ((p0 + p1) + p2) + ...; otherwise (SPLIT = 1) each
(g, c) fold runs over j = 0..NS-1 in order.  The template fuses the c loop
into the j loop (independent accumulators), tiles each warp's chunk through
its own shared-memory tile (all lanes read the same source record:
broadcast LDS.128), and register-blocks RB targets per thread so one staged
source serves RB x C accumulators; the compiler CSEs the per-pair work
shared by the C components (distance, rsqrt).  This template is emitted with fast math
(FMA contraction, MUFU rsqrt): parity is the tolerance of DESIGN.md (no
worse than the reference's own fp32 left fold, measured against fp64).
"""

from __future__ import annotations

from . import lir
from ._ref import nat
from .emit_cuda import GenericKernel, NatRenderer, Stage, ValueRenderer, kernel_head, py_expr
from .vec2 import NoVec2, Vec2

import os

# a block is SPLIT warps over the same 32*RB targets, warp w folding the w-th
# contiguous chunk of the sources: 1024 blocks x 16 warps for 131072 bodies,
# 32 resident warps per SM (the target count alone gives only ~7); measured
# on B200: SPLIT 1 / 4 / 8 / 16 -> 0.52 / 0.63 / 0.67 / 0.67 of FP32 peak
SPLIT = int(os.environ.get("RISE_ALLPAIRS_SPLIT", "16"))
RB = int(os.environ.get("RISE_ALLPAIRS_RB", "4"))  # targets per thread
# sources per warp tile, source-loop unroll and __launch_bounds__ min blocks
# per SM (0: none).  Measured at 131072 bodies (round 2, one B200):
#   JT 32, unroll 4, no min            0.684 of the FP32 peak (round-1 default)
#   min 1 (the compiler may use up to 128 registers: one 16-warp block per SM,
#   and a schedule that overlaps more of the r2 -> rsqrt -> scale chains)
#         unroll 4 / 8 / 16            0.686 / 0.691 / 0.691
#   min 1, JT 64, unroll 8 / 16 / 64   0.702 / 0.702 / 0.702   <- default
#   JT 64 without min 1                0.680; min 2 / 3-6        0.678 / 0.60-0.65
#   the next tile prefetched into registers during the fold: 0.696 (the
#   staging latency is not on the critical path); a constant-trip fold loop
#   for full tiles: no change
JT = int(os.environ.get("RISE_ALLPAIRS_JT", "64"))
UNROLL = int(os.environ.get("RISE_ALLPAIRS_UNROLL", "8"))
PACKED = os.environ.get("RISE_ALLPAIRS_PACKED", "1") == "1"  # two targets per FFMA2/FADD2/FMUL2
MINB = int(os.environ.get("RISE_ALLPAIRS_MINB", "1"))


def _split(body):
    """-> (cvar, C, acc, init, jloop, post) or None"""
    cvar, C = None, nat.Const(1)
    if isinstance(body, lir.For):
        cvar, C = body.var, body.bound
        body = body.body
        if not isinstance(C, nat.Const) or C.value > 8:
            return None
    if not (isinstance(body, lir.Alloc) and body.dims == () and body.space == "Private"):
        return None
    acc = lir.ScalarRef(body.name, body.ctype)
    stmts = body.body.stmts if isinstance(body.body, lir.Seq) else [body.body]
    if len(stmts) < 2:
        return None
    init, jloop, post = stmts[0], stmts[1], stmts[2:]
    if not (isinstance(init, lir.Assign) and init.target == acc and isinstance(jloop, lir.For)):
        return None
    for s in post:
        for t in lir.walk(s):
            if isinstance(t, (lir.For, lir.ParFor, lir.Alloc, lir.DoubleBuffer)):
                return None
    # the fold body may only write acc and its own private temporaries
    local = {s.name for s in lir.walk(jloop.body) if isinstance(s, lir.Alloc)}
    for s in lir.walk(jloop.body):
        if isinstance(s, (lir.ParFor, lir.DoubleBuffer, lir.Raw)):
            return None
        if isinstance(s, lir.Alloc) and s.space == "Global":
            return None
        if isinstance(s, lir.Assign):
            t = s.target
            if isinstance(t, lir.ScalarRef) and t != acc and t.name not in local:
                return None
            if isinstance(t, lir.Store) and t.buf not in local:
                return None
    return cvar, C, acc, init, jloop, post


def _fold_is_sum(body, acc):
    """True when the fold step is exactly `acc = acc + e` (e free of acc) and
    acc is written nowhere else: only then may the sources be split into
    chunks whose partial sums are added afterwards."""
    writes = [s for s in lir.walk(body) if isinstance(s, lir.Assign) and s.target == acc]
    if len(writes) != 1:
        return False
    def straight(s):  # statements reached through Seq / Alloc only (run once per j)
        yield s
        if isinstance(s, lir.Seq):
            for c in s.stmts:
                yield from straight(c)
        elif isinstance(s, lir.Alloc):
            yield from straight(s.body)

    if not any(s is writes[0] for s in straight(body)):
        return False
    v = writes[0].value
    if not (isinstance(v, lir.Bin) and v.op == "+" and v.ctype == "float"):
        return False
    if v.a == acc:
        other = v.b
    elif v.b == acc:
        other = v.a
    else:
        return False
    return acc not in set(lir.expr_scalars(other))


def _const_loop_bounds(stmt):
    out = {}
    for s in lir.walk(stmt):
        if isinstance(s, lir.For):
            out[s.var] = s.bound
    return out


def _source_stride(index, j, allowed_off_vars, bounds, cvar, C):
    """index = a*j + off with 0 <= off < a: returns a (int) or None."""
    zero = nat.normalize(nat.substitute(index, {j: nat.Const(0)}))
    one = nat.normalize(nat.substitute(index, {j: nat.Const(1)}))
    two = nat.normalize(nat.substitute(index, {j: nat.Const(2)}))
    a = nat.normalize(one - zero)
    if not isinstance(a, nat.Const) or a.value < 1:
        return None
    if not nat.equal(nat.normalize(two - zero), nat.Const(2 * a.value)):
        return None
    off_vars = nat.free_vars(zero)
    if not off_vars <= allowed_off_vars:
        return None
    # range of off over the constant loops
    lo = hi = nat.normalize(nat.substitute(zero, {v: nat.Const(0) for v in off_vars}))
    if not isinstance(lo, nat.Const):
        return None
    lo = hi = lo.value
    for v in off_vars:
        b = C if v == cvar else bounds.get(v)
        if not isinstance(b, nat.Const):
            return None
        z = {u: nat.Const(0) for u in off_vars}
        o = dict(z)
        o[v] = nat.Const(1)
        coef = nat.normalize(nat.substitute(zero, o) - nat.substitute(zero, z))
        if not isinstance(coef, nat.Const):
            return None
        span = coef.value * (b.value - 1)
        lo += min(0, span)
        hi += max(0, span)
    if lo < 0 or hi >= a.value:
        return None
    return a.value


def match(prog, stage, base_name, temps, exact, parallel_rows):
    loops, body = parallel_rows(stage)
    if loops is None or len(loops) != 1 or stage.kind != "grid":
        return None
    (gv, NT), = loops
    sp = _split(body)
    if sp is None:
        return None
    cvar, C, acc, init, jloop, post = sp
    j = jloop.var
    NS = jloop.bound
    if not nat.free_vars(NS) <= set(prog.nat_params):
        return None
    bounds = _const_loop_bounds(jloop.body)
    allowed_off = set(bounds) | ({cvar} if cvar else set())
    streams = {}  # buf -> stride
    for _t, value in lir.stmt_exprs(jloop.body):
        for ld in lir.expr_loads(value):
            if j not in nat.free_vars(ld.index):
                continue
            buf = prog.buffers[ld.buf]
            if buf.role != "input":
                return None
            a = _source_stride(ld.index, j, allowed_off, bounds, cvar, C)
            if a is None or streams.get(ld.buf, a) != a:
                return None
            streams[ld.buf] = a
    if not streams or any(prog.buffers[b].ctype != "float" for b in streams):
        return None
    s_list = sorted(streams.items())
    name = f"{base_name}_allpairs"
    r = NatRenderer(prog.clamps)
    fast = False  # fast math: FMA contraction + MUFU rsqrt

    # sources are staged as array-of-records: one record of REC floats per
    # source (e.g. x, y, z, m), 16-byte aligned, so a record is one LDS.128
    offsets, rec = {}, 0
    for buf, a in s_list:
        offsets[buf] = rec
        rec += a
    rec = -(-rec // 4) * 4 if rec > 2 else rec

    def hook(ld):
        if ld.buf in streams and j in nat.free_vars(ld.index):
            a = streams[ld.buf]
            off = nat.normalize(ld.index - nat.Var(j) * nat.Const(a))
            return f"rs_s[({j} - rs_j0) * {rec} + {offsets[ld.buf]} + ({r(off)})]"
        return None

    g = GenericKernel(prog, Stage("serial", jloop.body), "_", [], exact=fast)
    g.r = ValueRenderer(prog, exact=fast, load_hook=hook)
    step_lines = g.thread(jloop.body, 2)
    packed = PACKED and RB % 2 == 0 and acc.ctype == "float"
    step2_lines = None
    if packed:
        try:
            step2_lines = Vec2(prog, gv, lambda ld, _lane: hook(ld), exact=False,
                               names=("rs_ga", "rs_gb")).stmt(jloop.body, 2)
        except NoVec2:
            packed = False
    gp = GenericKernel(prog, Stage("serial", lir.Seq(list(post))), "_", [], exact=fast)
    post_lines = gp.thread(lir.Seq(list(post)), 3)
    vinit = ValueRenderer(prog, exact=fast)(init.value)
    Cv = C.value
    cdecl = f"const int {cvar}" if cvar else "const int rs_c_unused"
    split = SPLIT if _fold_is_sum(jloop.body, acc) else 1
    nthreads = 32 * split
    peer = int(getattr(prog, "peer_ranks", 0) or 0)
    extra = ["const unsigned long long* __restrict__ rs_peer"] if peer else []
    lines = kernel_head(prog, name, temps, launch_bounds=f"{nthreads}, {MINB}" if MINB else nthreads,
                        extra_params=extra)
    lines += [
        f"  constexpr int RS_NT = {r(NT)}, RS_NS = {r(NS)}, RS_JT = {JT}, RS_RB = {RB}, RS_C = {Cv};",
        f"  constexpr int RS_SPLIT = {split}, RS_CH = (RS_NS + RS_SPLIT - 1) / RS_SPLIT;",
    ]
    if peer:
        lines += [
            f"  constexpr int RS_RANKS = {peer}, RS_PER_RANK = RS_NS / RS_RANKS;",
        ]
    lines += [
        # one source tile per warp: the warps of a block fold disjoint source
        # chunks for the same targets, so a warp only ever syncs with itself
        f"  __shared__ __align__(16) float rs_sm[RS_SPLIT][RS_JT * {rec}];",
        "  const int rs_w = threadIdx.x >> 5, rs_l = threadIdx.x & 31;",
        "  float* const rs_s = rs_sm[rs_w];",
        "  const int rs_g0 = blockIdx.x * (32 * RS_RB) + rs_l;",
        "  int rs_j0 = 0;",
        f"  auto rs_step = [&](const int {gv}, {cdecl}, const int {j}, {acc.ctype} {acc.name}) -> {acc.ctype} {{",
    ]
    lines += step_lines
    lines += [
        f"    return {acc.name};",
        "  };",
    ]
    if packed:
        # the same step for two targets at once, in packed fp32x2 arithmetic
        lines.append(f"  auto rs_step2 = [&](const int rs_ga, const int rs_gb, {cdecl}, const int {j}, "
                     f"float2 {acc.name}) -> float2 {{")
        lines += step2_lines
        lines += [f"    return {acc.name};", "  };"]
    init_expr = vinit if split == 1 else f"(rs_w == 0 ? ({vinit}) : ({acc.ctype})0)"
    lines += [
        f"  {acc.ctype} rs_acc[RS_RB][RS_C];",
        "  int rs_gt[RS_RB];",
        "#pragma unroll",
        "  for (int rs_r = 0; rs_r < RS_RB; ++rs_r) {",
        f"    const int {gv} = min(rs_g0 + rs_r * 32, RS_NT - 1);",
        f"    rs_gt[rs_r] = {gv};",
        "#pragma unroll",
        "    for (int rs_c = 0; rs_c < RS_C; ++rs_c) {",
        f"      {cdecl} = rs_c;",
        f"      rs_acc[rs_r][rs_c] = {init_expr};",
        "    }",
        "  }",
        "  const int rs_jb = rs_w * RS_CH;",
        "  const int rs_je = RS_NS < rs_jb + RS_CH ? RS_NS : rs_jb + RS_CH;",
        "  for (rs_j0 = rs_jb; rs_j0 < rs_je; rs_j0 += RS_JT) {",
        "    const int rs_jn = rs_je - rs_j0 < RS_JT ? rs_je - rs_j0 : RS_JT;",
        "    __syncwarp();",
    ]
    if peer:
        # the sources live in the R ranks' blocks (peer memory over NVLink):
        # a tile never straddles two blocks (preconditions), so its records
        # are read straight from the owning rank — the all-gather is fused
        # into the staging of the fold
        lines += [
            "    const int rs_rank = rs_j0 / RS_PER_RANK, rs_jl = rs_j0 - rs_rank * RS_PER_RANK;",
        ]
    for k, (buf, a) in enumerate(s_list):
        src = (f"reinterpret_cast<const float*>(rs_peer[{k} * RS_RANKS + rs_rank])[{a} * rs_jl + rs_e]" if peer
               else f"{buf}[{a} * rs_j0 + rs_e]")
        lines += [
            "#pragma unroll 4",
            f"    for (int rs_e = rs_l; rs_e < rs_jn * {a}; rs_e += 32)",
            f"      rs_s[(rs_e / {a}) * {rec} + {offsets[buf]} + rs_e % {a}] = {src};",
        ]
    lines += [
        "    __syncwarp();",
        f"#pragma unroll {UNROLL}",
        "    for (int rs_jj = 0; rs_jj < rs_jn; ++rs_jj) {",
    ]
    if packed:
        lines += [
            "#pragma unroll",
            "      for (int rs_p = 0; rs_p < RS_RB / 2; ++rs_p) {",
            "#pragma unroll",
            "        for (int rs_c = 0; rs_c < RS_C; ++rs_c) {",
            "          float2 rs_a2 = make_float2(rs_acc[2 * rs_p][rs_c], rs_acc[2 * rs_p + 1][rs_c]);",
            "          rs_a2 = rs_step2(rs_gt[2 * rs_p], rs_gt[2 * rs_p + 1], rs_c, rs_j0 + rs_jj, rs_a2);",
            "          rs_acc[2 * rs_p][rs_c] = rs_a2.x;",
            "          rs_acc[2 * rs_p + 1][rs_c] = rs_a2.y;",
            "        }",
            "      }",
        ]
    else:
        lines += [
            "#pragma unroll",
            "      for (int rs_r = 0; rs_r < RS_RB; ++rs_r) {",
            "#pragma unroll",
            "        for (int rs_c = 0; rs_c < RS_C; ++rs_c)",
            "          rs_acc[rs_r][rs_c] = rs_step(rs_gt[rs_r], rs_c, rs_j0 + rs_jj, rs_acc[rs_r][rs_c]);",
            "      }",
        ]
    lines += ["    }", "  }"]
    if split > 1:
        add = "__fadd_rn" if acc.ctype == "float" else ""
        lines += [
            # chunk partials meet in shared memory and are added in chunk order
            f"  __shared__ {acc.ctype} rs_part[RS_SPLIT - 1][RS_RB * RS_C][32];",
            "  if (rs_w > 0) {",
            "#pragma unroll",
            "    for (int rs_r = 0; rs_r < RS_RB; ++rs_r)",
            "#pragma unroll",
            "      for (int rs_c = 0; rs_c < RS_C; ++rs_c)",
            "        rs_part[rs_w - 1][rs_r * RS_C + rs_c][rs_l] = rs_acc[rs_r][rs_c];",
            "  }",
            "  __syncthreads();",
            "  if (rs_w != 0) return;",
            "  for (int rs_q = 0; rs_q < RS_SPLIT - 1; ++rs_q) {",
            "#pragma unroll",
            "    for (int rs_r = 0; rs_r < RS_RB; ++rs_r)",
            "#pragma unroll",
            "      for (int rs_c = 0; rs_c < RS_C; ++rs_c)",
            f"        rs_acc[rs_r][rs_c] = {add}(rs_acc[rs_r][rs_c], rs_part[rs_q][rs_r * RS_C + rs_c][rs_l]);",
            "  }",
        ]
    lines += [
        "#pragma unroll",
        "  for (int rs_r = 0; rs_r < RS_RB; ++rs_r) {",
        f"    const int {gv} = rs_g0 + rs_r * 32;",
        f"    if ({gv} < RS_NT) {{",
        "#pragma unroll",
        "      for (int rs_c = 0; rs_c < RS_C; ++rs_c) {",
        f"        {cdecl} = rs_c;",
        f"        {acc.ctype} {acc.name} = rs_acc[rs_r][rs_c];",
    ]
    lines += post_lines
    lines += ["      }", "    }", "  }", "}"]
    plan = {
        "name": name,
        "kind": "allpairs",
        "targets": py_expr(NT),
        "per_block": 32 * RB,
        "block": nthreads,
        "split": split,
        **({"peer_ranks": peer, "peer_streams": [b for b, _a in s_list],
            "extra_args": [{"kind": "peer_table"}]} if peer else {}),
        "fmad": True,
        "order": ("preserved-fold" if split == 1 else f"{split} contiguous source chunks, added in chunk order")
        + ", fast-math",
        "pre": ([f"({py_expr(NS)}) % {peer} == 0", f"(({py_expr(NS)}) // {peer}) % {JT} == 0",
                 f"(({py_expr(NS)}) // {split}) % {JT} == 0", f"({py_expr(NS)}) % {split} == 0"] if peer else []),
    }
    return "\n".join(lines) + "\n", plan


def launch(st, nats, sm):
    from .emit_cuda import eval_py

    nt = eval_py(st["targets"], nats)
    return (max(1, -(-nt // st["per_block"])), 1, 1), (st["block"], 1, 1), 0, (1, 1, 1)
