"""`stencil2d` template: a 2-D parallel map whose body reads a 2-D array
through clamped neighbourhood indices (padClamp2D + slide2D programs).

Matches a stage whose parallel loops collapse to exactly two variables
(r < R, c < C) and in which every load of some 2-D input A has per-dimension
indices  clamp(r + o0, H-1)  and  clamp(c + o1, W-1),  where o0 / o1 are
affine in sequential loop variables with constant bounds (the window
offsets).  The offsets' ranges [omin, omax] give the halo.

Order: PRESERVED.  The body is the generic emitter's code for the program's
own loop nest (row sums, then the fold of the row sums, with the
round-to-nearest intrinsics); only the loads of A are redirected.
Bit-identical to the reference's semantics.

Data movement:
* a block computes a TR x TC = 32 x 256 output tile (64 x 4 threads, each
  thread RPT = 8 rows x CPT = 4 adjacent columns; 1-KiB row segments keep
  the DRAM streams long: 0.80 of the copy peak against 0.77 for 64 x 128);
* the tile's input footprint (rows + halo, columns + halo, left edge padded
  to a 16-byte boundary) is staged into shared memory by the bulk-copy
  engine: ONE 2-D TMA load when a staged row fits a TMA box (<= 256
  elements), else one 1-D bulk copy per staged row (`rowcopy`, the default
  264-column footprint); border tiles then get the padClamp values by an
  in-shared-memory fix-up, so no per-access clamp remains in the compute;
* each thread copies its (RPT + halo) x (CPT + halo) window from shared
  memory into registers (LDS.128 for the aligned middle columns), and the
  body's loads of A become constant-indexed register reads after unrolling
  — one staged value serves every output of the window that uses it.
"""

from __future__ import annotations

from . import lir
from ._ref import nat
from .emit_cuda import GenericKernel, NatRenderer, Stage, ValueRenderer, kernel_head, py_expr

import os  # noqa: E402

# threads along a row (4 adjacent columns each).  Measured (8192², 3 blocks
# per SM, round-robin inputs): 32 -> 64 x 128 tiles 0.77, 64 -> 32 x 256
# tiles 0.80, 128 -> 16 x 512 tiles 0.75 (the row halo grows)
TX = int(os.environ.get("RISE_STENCIL_TX", "64"))
TY = int(os.environ.get("RISE_STENCIL_TY", str(256 // TX)))
RPT = int(os.environ.get("RISE_STENCIL_RPT", "8"))  # output rows per thread
CPT = 4  # adjacent output columns per thread
TR, TC = TY * RPT, TX * CPT

# persistent blocks per SM (each holds two 36 KB stages); overridable for sweeps
BLOCKS_PER_SM = int(os.environ.get("RISE_STENCIL_BPS", "3"))
# full tiles leave through shared memory and one TMA tile store, or one bulk
# store per row in rowcopy mode (else 16-byte STGs)
TMA_STORE = os.environ.get("RISE_STENCIL_TMA_STORE", "1") == "1"
STAGES = int(os.environ.get("RISE_STENCIL_STAGES", "2"))  # ring depth per block (measured: 2 x 3 blocks/SM 0.82 > 3 x 2 0.78 > 4 x 1 0.77)


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
    zero = {v: nat.Const(0) for v in nat.free_vars(off)}
    lo = nat.normalize(nat.substitute(off, zero))
    if not isinstance(lo, nat.Const):
        return None
    lo = hi = lo.value
    for v in nat.free_vars(off):
        b = loop_bounds.get(v)
        if b is None or not isinstance(b, nat.Const) or b.value < 1:
            return None
        one = dict(zero)
        one[v] = nat.Const(1)
        two = dict(zero)
        two[v] = nat.Const(2)
        coef = nat.normalize(nat.substitute(off, one) - nat.substitute(off, zero))
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
    tiled = {}  # buf -> [omin0, omax0, omin1, omax1]
    for _t, value in lir.stmt_exprs(body):
        for ld in lir.expr_loads(value):
            if not any(v in prog.clamps for v in nat.free_vars(ld.index)):
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
    if len(tiled) != 1 or any(prog.buffers[b].ctype != "float" for b in tiled):
        return None
    (abuf, (o0lo, o0hi, o1lo, o1hi)), = tiled.items()
    if not (o0lo <= 0 <= o0hi and o1lo <= 0 <= o1hi) or o0hi - o0lo > 8 or o1hi - o1lo > 8:
        return None
    A = prog.buffers[abuf]
    name = f"{base_name}_stencil"
    r = NatRenderer(prog.clamps)
    hr = o0hi - o0lo  # halo rows
    hcl, hcr = -o1lo, o1hi  # halo columns left / right
    lp = -(-hcl // 4) * 4  # left pad, keeps the thread's columns 16-byte aligned
    sw = -(-(lp + TC + hcr) // 4) * 4  # staged row width (multiple of 16 bytes)
    sr = TR + hr  # staged rows
    # staged rows wider than a TMA box (<= 256 elements) arrive as one 1-D
    # bulk copy per row and leave as one bulk store per row
    rowcopy = sw > 256 or os.environ.get("RISE_STENCIL_ROWCOPY", "0") == "1"
    wr, wc = RPT + hr, CPT + hcl + hcr  # register window

    # small row/column-invariant inputs (e.g. the 3x3 weights) live in registers
    small = {}
    for _t, value in lir.stmt_exprs(body):
        for ld in lir.expr_loads(value):
            b = prog.buffers[ld.buf]
            if ld.buf == abuf or b.role != "input" or rv in nat.free_vars(ld.index) or cv in nat.free_vars(ld.index):
                continue
            size = nat.Const(1)
            for d in b.dims:
                size = size * d
            size = nat.normalize(size)
            if isinstance(size, nat.Const) and size.value <= 64:
                small[ld.buf] = size.value

    def hook(ld):
        if ld.buf in small:
            return f"rs_p_{ld.buf}[{r(ld.index)}]"
        if ld.buf != abuf:
            return None
        e0, e1 = ld.indices
        off0 = nat.normalize(prog.clamps[e0.name][0] - nat.Var(rv))
        off1 = nat.normalize(prog.clamps[e1.name][0] - nat.Var(cv))
        return f"rs_v[rs_k + ({r(off0)}) + {-o0lo}][rs_q + ({r(off1)}) + {hcl}]"

    g = GenericKernel(prog, Stage("serial", body), "_", [], exact)
    g.r = ValueRenderer(prog, exact, load_hook=hook)
    body_lines = g.thread(body, 4)
    # the output tile always fits a TMA box ([TR][TC], TC <= 256): rows staged
    # by bulk copies still leave by one 2-D TMA store (RISE_STENCIL_OMAP=0: one
    # bulk store per row; measured 0.895 -> 0.903 of HBM with the tile store)
    omap = not rowcopy or os.environ.get("RISE_STENCIL_OMAP", "1") == "1"
    pair_lines, store_pre, ostore = _pair_body(prog, body, rv, cv, abuf, small, hook, exact, r, TMA_STORE,
                                               rowcopy and not omap)
    tma_store = ostore is not None
    hdim = r(nat.normalize(A.dims[0] - nat.Const(1)))
    wdim = r(nat.normalize(A.dims[1] - nat.Const(1)))
    params = [] if rowcopy else ["const __grid_constant__ rs_tmap rs_map"]
    if tma_store and omap:
        params.append("const __grid_constant__ rs_tmap rs_omap")
    peer_halo = bool(getattr(prog, "peer_halo", False))
    ht, hb = -o0lo, o0hi  # rows of halo above / below the band
    row_pass = [
        "        if (rs_y < rs_ylo) rs_tile[rs_e] = rs_tile[rs_ylo * RS_SW + rs_x];",
        "        else if (rs_y > rs_yhi) rs_tile[rs_e] = rs_tile[rs_yhi * RS_SW + rs_x];",
    ]
    if peer_halo:
        # multi-GPU row bands: the rows padClamp would invent above / below
        # this band are the neighbours' edge rows, read in place (peer
        # pointers over NVLink; NULL at the image's real edges = clamp) —
        # the halo exchange fused into the stencil's border-tile staging
        params += ["const float* __restrict__ rs_halo_top", "const float* __restrict__ rs_halo_bot"]
        row_pass = [
            "        const int rs_gc = rs_tc0 + rs_x;  // image column of the cell",
            "        const bool rs_cin = rs_gc >= 0 && rs_gc < RS_W;",
            "        if (rs_y < rs_ylo) rs_tile[rs_e] = rs_halo_top != nullptr && rs_cin",
            f"            ? rs_halo_top[(rs_tr0 + rs_y + {ht}) * RS_W + rs_gc] : rs_tile[rs_ylo * RS_SW + rs_x];",
            "        else if (rs_y > rs_yhi) rs_tile[rs_e] = rs_halo_bot != nullptr && rs_cin",
            "            ? rs_halo_bot[(rs_tr0 + rs_y - RS_H) * RS_W + rs_gc] : rs_tile[rs_yhi * RS_SW + rs_x];",
        ]
    lines = kernel_head(prog, name, temps, launch_bounds=f"{TX * TY}, {BLOCKS_PER_SM}", extra_params=params)
    lines += [
        f"  constexpr int RS_R = {r(R)}, RS_C = {r(C)};",
        f"  constexpr int RS_H = {r(A.dims[0])}, RS_W = {r(A.dims[1])};",
        f"  constexpr int RS_SR = {sr}, RS_SW = {sw};",
        "  constexpr int RS_STAGE = (RS_SR * RS_SW + 31) / 32 * 32;  // stages stay 128-byte aligned (TMA)",
        f"  constexpr int RS_NSTAGE = {STAGES};",
        f"  constexpr int RS_NTX = (RS_C + {TC - 1}) / {TC}, RS_NTY = (RS_R + {TR - 1}) / {TR};",
        "  constexpr int RS_NTILES = RS_NTX * RS_NTY;",
        "  extern __shared__ __align__(128) unsigned char rs_dsmem[];",
        "  float* rs_buf = reinterpret_cast<float*>(rs_dsmem + ((128u - (rs_smem_addr(rs_dsmem) & 127u)) & 127u));",
        "  unsigned long long* rs_bar = reinterpret_cast<unsigned long long*>(rs_buf + RS_NSTAGE * RS_STAGE);",
        "  const int rs_tid = threadIdx.y * blockDim.x + threadIdx.x;",
        "  // tile t -> (rs_r0, rs_c0); interior tiles arrive by TMA, border tiles by clamped loads",
        "  auto rs_origin = [&](int t, int& r0, int& c0) {",
        f"    r0 = (t / RS_NTX) * {TR}; c0 = (t % RS_NTX) * {TC};",
        "  };",
        "  auto rs_is_interior = [&](int r0, int c0) {",
        f"    const int tr0 = r0 + ({o0lo}), tc0 = c0 - {lp};",
        "    return tr0 >= 0 && tr0 + RS_SR <= RS_H && tc0 >= 0 && tc0 + RS_SW <= RS_W;",
        "  };",
        "  auto rs_issue = [&](int t, int s) {  // thread 0 only; border tiles too (out-of-range cells arrive as 0)",
        "    int r0, c0;",
        "    rs_origin(t, r0, c0);",
        "    rs_fence_proxy_async();  // earlier generic-proxy accesses of this stage precede the TMA write",
    ] + ([
        "    rs_mbar_arrive_expect_tx(&rs_bar[s], (unsigned)(RS_SR * RS_SW * 4));",
        f"    rs_tma_load_2d(rs_buf + s * RS_STAGE, &rs_map, c0 - {lp}, r0 + ({o0lo}), &rs_bar[s]);",
    ] if not rowcopy else [
        "    // one bulk copy per staged row, in-range cells only (the clamp fix-up fills the rest)",
        f"    const int tr0 = r0 + ({o0lo}), tc0 = c0 - {lp};",
        "    const int cs = tc0 < 0 ? 0 : tc0, ce = tc0 + RS_SW > RS_W ? RS_W : tc0 + RS_SW;",
        "    const int ys = tr0 < 0 ? -tr0 : 0, ye = tr0 + RS_SR > RS_H ? RS_H - tr0 : RS_SR;",
        "    rs_mbar_arrive_expect_tx(&rs_bar[s], (unsigned)((ye - ys) * (ce - cs) * 4));",
        "    for (int y = ys; y < ye; ++y)",
        f"      rs_bulk_g2s(rs_buf + s * RS_STAGE + y * RS_SW + (cs - tc0), {abuf} + (tr0 + y) * RS_W + cs,",
        "                  (unsigned)((ce - cs) * 4), &rs_bar[s]);",
    ]) + [
        "  };",
        "  if (rs_tid == 0) {",
        "    for (int rs_q = 0; rs_q < RS_NSTAGE; ++rs_q) rs_mbar_init(&rs_bar[rs_q], 1);",
        "    rs_fence_barrier_init();",
        "    for (int rs_q = 0; rs_q < RS_NSTAGE - 1; ++rs_q)",
        "      if ((int)blockIdx.x + rs_q * (int)gridDim.x < RS_NTILES) rs_issue(blockIdx.x + rs_q * gridDim.x, rs_q);",
        "  }",
        "  __syncthreads();",
    ]
    for buf, size in sorted(small.items()):
        lines += [
            f"  float rs_p_{buf}[{size}];",
            "#pragma unroll",
            f"  for (int rs_e = 0; rs_e < {size}; ++rs_e) rs_p_{buf}[rs_e] = __ldg({buf} + rs_e);",
        ]
    lines += [
        "  int rs_it = 0;",
        "  for (int rs_t = blockIdx.x; rs_t < RS_NTILES; rs_t += gridDim.x, ++rs_it) {",
        "    const int rs_s = rs_it % RS_NSTAGE;",
        "    int rs_r0, rs_c0;",
        "    rs_origin(rs_t, rs_r0, rs_c0);",
        f"    const int rs_tr0 = rs_r0 + ({o0lo}), rs_tc0 = rs_c0 - {lp};",
        "    float* rs_tile = rs_buf + rs_s * RS_STAGE;",
        "    // prefetch NSTAGE-1 tiles ahead into the stage the previous tile used (freed by the barrier",
        "    // that ended it)",
        "    if (rs_tid == 0 && rs_t + (RS_NSTAGE - 1) * (int)gridDim.x < RS_NTILES) {",
        "      rs_bulk_wait_read_all();  // that stage staged the previous tile's output (TMA store)" if tma_store else "",
        "      rs_issue(rs_t + (RS_NSTAGE - 1) * gridDim.x, (rs_it + RS_NSTAGE - 1) % RS_NSTAGE);",
        "    }",
        "    rs_mbar_wait(&rs_bar[rs_s], (unsigned)((rs_it / RS_NSTAGE) & 1));",
        "    if (!rs_is_interior(rs_r0, rs_c0)) {",
        "      // padClamp: every out-of-range staged cell takes the value of the nearest in-range",
        "      // cell, which the same box holds (the box always contains an in-range row and column)",
        "      const int rs_ylo = rs_tr0 < 0 ? -rs_tr0 : 0, rs_xlo = rs_tc0 < 0 ? -rs_tc0 : 0;",
        f"      const int rs_yhi = {hdim} - rs_tr0, rs_xhi = {wdim} - rs_tc0;  // last in-range staged row / column",
    ] + _fixup_lines(row_pass, TX * TY) + [
        "    }",
        "    // this thread's register window (tile rows ty*RPT.., columns lp + tx*CPT - hcl..)",
        f"    float rs_v[{wr}][{wc}];",
        "#pragma unroll",
        f"    for (int rs_y = 0; rs_y < {wr}; ++rs_y) {{",
        f"      const float* rs_row = rs_tile + (threadIdx.y * {RPT} + rs_y) * RS_SW + {lp} + threadIdx.x * {CPT};",
        "      const float4 rs_mid = *reinterpret_cast<const float4*>(rs_row);",
    ]
    for k in range(hcl):
        lines.append(f"      rs_v[rs_y][{k}] = rs_row[{k - hcl}];")
    lines += [
        f"      rs_v[rs_y][{hcl}] = rs_mid.x; rs_v[rs_y][{hcl + 1}] = rs_mid.y;",
        f"      rs_v[rs_y][{hcl + 2}] = rs_mid.z; rs_v[rs_y][{hcl + 3}] = rs_mid.w;",
    ]
    for k in range(hcr):
        lines.append(f"      rs_v[rs_y][{hcl + CPT + k}] = rs_row[{CPT + k}];")
    lines += [
        "    }",
        "    __syncthreads();  // the stage may be refilled once every thread holds its window",
    ]
    for guarded in (False, True):
        if not guarded:
            lines.append(f"    if (rs_r0 + {TR} <= RS_R && rs_c0 + {TC} <= RS_C) {{")
            if pair_lines is not None:
                # full tile: two adjacent columns per packed fp32x2 body, a
                # row's CPT = 4 outputs leave as one 16-byte store
                lines += pair_lines
                continue
        else:
            lines.append("    } else {")
        lines += [
            "#pragma unroll",
            f"    for (int rs_k = 0; rs_k < {RPT}; ++rs_k) {{",
            "#pragma unroll",
            f"      for (int rs_q = 0; rs_q < {CPT}; ++rs_q) {{",
            f"        const int {rv} = rs_r0 + threadIdx.y * {RPT} + rs_k;",
            f"        const int {cv} = rs_c0 + threadIdx.x * {CPT} + rs_q;",
            f"        if ({'true' if not guarded else f'{rv} < RS_R && {cv} < RS_C'}) {{",
        ]
        lines += ["  " + x for x in body_lines]
        lines += ["        }", "      }", "    }"]
    lines += ["    }", "  }"]
    if tma_store:
        lines.append("  if (rs_tid == 0) rs_bulk_wait_all();  // the last tile's store has left shared memory")
    lines += ["}"]
    lines = [x for x in lines if x != ""]
    smem = STAGES * (-(-(sr * sw) // 32) * 32) * 4 + 8 * STAGES + 128
    plan = {
        "name": name,
        "kind": "stencil2d",
        "rows": py_expr(R),
        "cols": py_expr(C),
        "tile": [TR, TC],
        "block": [TX, TY],
        "smem": smem,
        "blocks_per_sm": BLOCKS_PER_SM,
        "fmad": False,
        "order": "preserved",
        "pre": [f"({py_expr(A.dims[1])}) % 4 == 0", f"({py_expr(R)}) * ({py_expr(C)}) > 0"] + store_pre,
        "packed": pair_lines is not None,
        "extra_args": [] if rowcopy else [{"kind": "tma2d", "buf": abuf, "offset": "0",
                                           "dims": [py_expr(A.dims[1]), py_expr(A.dims[0])],
                                           "pitch": py_expr(A.dims[1]), "box": [sw, sr], "swizzle": 0}],
    }
    if rowcopy:
        plan["rowcopy"] = True
    if tma_store and omap:
        row_coef, const = ostore
        plan["extra_args"].append({"kind": "tma2d", "buf": prog.output.name, "offset": py_expr(const),
                                   "dims": [py_expr(C), py_expr(R)], "pitch": py_expr(row_coef),
                                   "box": [TC, TR], "swizzle": 0})
        plan["tma_store"] = True
    if peer_halo:  # (kernel parameter order: [rs_map, [rs_omap]], rs_halo_top, rs_halo_bot)
        plan["peer_halo"] = True
        plan["halo_rows"] = [ht, hb]
        plan["extra_args"] += [{"kind": "peer_ptr", "name": "rs_halo_top"}, {"kind": "peer_ptr", "name": "rs_halo_bot"}]
    return "\n".join(lines) + "\n", plan


def _pair_body(prog, body, rv, cv, abuf, small, hook, exact, r, tma_store, rowcopy=False):
    """Packed fp32x2 version of the body for output columns (q, q + 1):
    (lines of the full-tile compute, extra preconditions, (row pitch, offset)
    of the output when it leaves by TMA store else None), or (None, [], None)."""
    from .vec2 import NoVec2, Vec2

    stored = []

    def hook2(ld, lane):
        h = hook(ld)
        if h is None or ld.buf in small:
            return h
        return h.replace("rs_q +", "rs_qa +" if lane == 0 else "rs_qb +")

    def store_hook(t, value):
        if t.buf != prog.output.name or stored:
            return None
        idx = nat.normalize(t.index)
        z = {cv: nat.Const(0), rv: nat.Const(0)}
        at = lambda a, b: nat.normalize(nat.substitute(idx, {rv: nat.Const(a), cv: nat.Const(b)}))  # noqa: E731
        base = nat.normalize(nat.substitute(idx, {cv: nat.Const(0)}))
        one = nat.normalize(at(0, 1) - at(0, 0))
        if not (isinstance(one, nat.Const) and one.value == 1) or cv in nat.free_vars(base):
            return None
        stored.append((base, nat.normalize(at(1, 0) - at(0, 0)), nat.normalize(nat.substitute(idx, z))))
        return [f"rs_o2 = {value};"]

    try:
        v = Vec2(prog, cv, hook2, exact=exact, store_hook=store_hook)
        blines = v.stmt(body, 4)
    except NoVec2:
        return None, [], None
    if len(stored) != 1:
        return None, [], None
    base, row_coef, const = stored[0]
    if nat.free_vars(row_coef) - set(prog.nat_params) or nat.free_vars(const) - set(prog.nat_params):
        return None, [], None
    pre = [f"({py_expr(row_coef)}) % 4 == 0", f"({py_expr(const)}) % 4 == 0"]
    out = prog.output.name
    lines = [
        "    auto rs_pair = [&](const int rs_k, const int rs_qa, const int rs_qb) -> float2 {",
        f"      const int {rv} = rs_r0 + threadIdx.y * {RPT} + rs_k;",
        f"      const int rs_la = rs_c0 + threadIdx.x * {CPT} + rs_qa, rs_lb = rs_c0 + threadIdx.x * {CPT} + rs_qb;",
        "      float2 rs_o2;",
    ]
    lines += blines
    lines += [
        "      return rs_o2;",
        "    };",
        "#pragma unroll",
        f"    for (int rs_k = 0; rs_k < {RPT}; ++rs_k) {{",
        f"      const int {rv} = rs_r0 + threadIdx.y * {RPT} + rs_k;",
        "      const float2 rs_lo = rs_pair(rs_k, 0, 1), rs_hi = rs_pair(rs_k, 2, 3);",
    ]
    if tma_store:
        # the stage is free once every thread holds its window: stage the
        # output tile there ([TR][TC], conflict-free STS.128) for one TMA store
        lines += [
            f"      *reinterpret_cast<float4*>(&rs_tile[(threadIdx.y * {RPT} + rs_k) * {TC} + threadIdx.x * {CPT}]) = "
            "make_float4(rs_lo.x, rs_lo.y, rs_hi.x, rs_hi.y);",
            "    }",
            "    rs_fence_proxy_async();  // the generic-proxy writes precede the TMA read",
            "    __syncthreads();",
            "    if (rs_tid == 0) {",
        ] + ([
            "      rs_tma_store_2d(&rs_omap, rs_c0, rs_r0, rs_tile);",
        ] if not rowcopy else [
            f"      for (int rs_y = 0; rs_y < {TR}; ++rs_y)  // one bulk store per output row",
            f"        rs_bulk_s2g({out} + ({r(const)}) + (rs_r0 + rs_y) * ({r(row_coef)}) + rs_c0, rs_tile + rs_y * {TC}, {TC * 4}u);",
        ]) + [
            "      rs_bulk_commit();",
            "    }",
        ]
        return lines, pre, (row_coef, const)
    lines += [
        f"      *reinterpret_cast<float4*>(&{out}[({r(base)}) + rs_c0 + threadIdx.x * {CPT}]) = "
        "make_float4(rs_lo.x, rs_lo.y, rs_hi.x, rs_hi.y);",
        "    }",
    ]
    return lines, pre, None


def launch(st, nats, sm):
    from .emit_cuda import eval_py

    rows = eval_py(st["rows"], nats)
    cols = eval_py(st["cols"], nats)
    tr, tc = st["tile"]
    tiles = -(-cols // tc) * -(-rows // tr)
    # Persistent, tile-strided: block b takes tiles b, b + G, b + 2G, ...  G is
    # kept ≡ 2 (mod 4) and ~10 % under the resident maximum: with G a multiple
    # of the strips per band (32 at 8192²) every block walks one column strip
    # in band steps of a power-of-two pitch and the blocks pile onto the same
    # HBM channels — measured at 8192² with 444 slots (round 1): G = 416 0.49,
    # 432 0.63, 440 0.73, 444 0.80, 442 0.84, 426 0.875, 418 0.878 of the copy
    # peak; with the halo-only border fix-up and the TMA tile store (round 2,
    # conv_fix_r02c.txt, conv_grid_r02c.txt): 382 0.925, 390 0.914, 394
    # 0.92-0.924, 398 0.9245-0.9247, 402 0.914-0.923, 406 0.908-0.922, 410
    # 0.89, 414 0.908, 418 0.896, 422-430 0.88.
    slots = sm * st.get("blocks_per_sm", 2)
    grid = (int(slots * 0.895) // 4) * 4 + 2 if slots >= 8 else slots
    grid = int(os.environ.get("RISE_STENCIL_GRID", "0")) or grid  # (probe: explicit persistent grid)
    grid = max(1, min(tiles, grid))
    return (grid, 1, 1), (st["block"][0], st["block"][1], 1), st.get("smem", 0), (1, 1, 1)



def _fixup_lines(row_pass, nt):
    """The padClamp fix-up of a border tile's staged footprint, visiting only
    the out-of-range cells: the rows outside [ylo, yhi] (full width), then
    the columns outside [xlo, xhi] (every row), so corner cells end up
    clamped in both dimensions.  (The round-1 form scanned the whole
    footprint twice: strong-scaled bands 0.73 / 0.59 / 0.45 -> 0.77 / 0.67 /
    0.57 of their N = 1 rate at 2 / 4 / 8 ranks, profiles/conv_fix_r02c.txt.)"""
    return [
        "      const int rs_na = rs_ylo, rs_nb = rs_yhi < RS_SR - 1 ? RS_SR - 1 - rs_yhi : 0;",
        f"      for (int rs_q = rs_tid; rs_q < (rs_na + rs_nb) * RS_SW; rs_q += {nt}) {{",
        "        const int rs_k = rs_q / RS_SW, rs_x = rs_q - rs_k * RS_SW;",
        "        const int rs_y = rs_k < rs_na ? rs_k : rs_yhi + 1 + (rs_k - rs_na), rs_e = rs_y * RS_SW + rs_x;",
        *row_pass,
        "      }",
        "      __syncthreads();",
        "      const int rs_ca = rs_xlo, rs_nc = rs_ca + (rs_xhi < RS_SW - 1 ? RS_SW - 1 - rs_xhi : 0);",
        f"      for (int rs_q = rs_tid; rs_q < RS_SR * rs_nc; rs_q += {nt}) {{",
        "        const int rs_y = rs_q / rs_nc, rs_k = rs_q - rs_y * rs_nc;",
        "        const int rs_x = rs_k < rs_ca ? rs_k : rs_xhi + 1 + (rs_k - rs_ca);",
        "        rs_tile[rs_y * RS_SW + rs_x] = rs_tile[rs_y * RS_SW + (rs_k < rs_ca ? rs_xlo : rs_xhi)];",
        "      }",
        "      __syncthreads();",
    ]
