"""`rowfold` template: a parallel map over rows, each row a sequential fold.

Matches (after the parallel loops are collapsed into a flat row index f):

    for each row f (parallel):            # parForGlobal chain, or
        acc = INIT                        # parForWorkGroup > parForLocal
        for j < K:  acc = STEP(acc, A1[base1(f) + j], ..., X1[c + j], ...)
        POST(acc)                         # e.g. output[f] = acc

where every j-dependent load is unit-stride in j: `row streams` (base
depends on the row, affine in f: base = c0 + f * pitch) and `shared streams`
(base independent of the row, e.g. the vector x of gemv).

Order: PRESERVED.  One thread folds one row in j order with the program's own
STEP expression (rendered with the round-to-nearest intrinsics), so results
are bit-identical to the reference's sequential semantics.

Data movement (the part the template adds): a ring of RS_STAGES shared-memory
stages.  Per stage and row stream, the TMA engine loads RS_KT/32 boxes of
[32 rows x 32 floats] from a 2-D tensor map (rows = f, inner = j) with the
128-byte swizzle, so lane l reading row l, 16-byte chunk c touches physical
chunk c ^ (l & 7): conflict-free LDS.128.  Shared streams arrive by 1-D bulk
copy.  One elected lane arms the stage's mbarrier with the expected bytes and
issues every copy (a handful of TMA instructions per stage instead of one
bulk copy per row); the warp consumes stage t while stages t+1.. are in
flight.  Block = one warp = 32 rows (16 or 8 for short matrices: rows_per_block).
"""

from __future__ import annotations

from . import lir
from ._ref import nat
from .emit_cuda import NatRenderer, ValueRenderer, kernel_head, py_expr

import os  # noqa: E402

ROWS = int(os.environ.get("RISE_ROWFOLD_ROWS", "0"))  # rows per block (8, 16 or 32); 0 = by row count

KT = int(os.environ.get("RISE_ROWFOLD_KT", "256"))  # columns per stage (KT/32 TMA boxes of 32 columns)
# measured (gemv 8192², L2 flushed, 32-row blocks): 128x6 0.835, 256x2 0.855, 512x2 0.65; (round-robin
# inputs, 28-row blocks, two passes): 256x2 0.924-0.929, 256x3 0.936-0.939 (chunked dot 0.563 -> 0.583)
# ring depth: 0 = as many stages as the block's shared-memory budget holds,
# up to MAX_STAGES.  A stage's fold is latency-bound (one dependent add per
# column per lane: 256 columns ~ 0.5 us), so the ring must reach ~ 2-3 us
# ahead to cover DRAM latency: 3 stages at 8192 rows (32-row boxes, 33 KiB
# stages), 6 at 4096, 12 at <= 2048 (row bands of strong-scaled gemv)
STAGES = int(os.environ.get("RISE_ROWFOLD_STAGES", "0"))
MAX_STAGES = int(os.environ.get("RISE_ROWFOLD_MAX_STAGES", "12"))
MIN_ROWS = int(os.environ.get("RISE_ROWFOLD_MIN_ROWS", "4"))
# shared-memory reads issued this many 4-column chunks ahead of their use
PF = int(os.environ.get("RISE_ROWFOLD_PF", "4"))
SM_COUNT = 148
# split rows (reassociating, deterministic): a row's fold is a dependent
# chain of K adds (~7 cycles each with one warp per SM sub-partition, about
# 31 us at K = 8192 — tools/probe_chain.cu), so when there are fewer rows
# than it takes to fill the GPU (strong-scaled row bands) each row is folded
# as S contiguous column chunks by S adjacent lanes and the chunk partials
# are added in chunk order: S = the smallest power of two <= 32 with
# rows * S >= SPLIT_TARGET, for K >= SPLIT_MIN_K.  Only under
# emit_cuda(reassociate=True) (the default) and only for a sum fold.
SPLIT_TARGET = int(os.environ.get("RISE_ROWFOLD_SPLIT_TARGET", "8192"))
SPLIT_MIN_K = int(os.environ.get("RISE_ROWFOLD_SPLIT_MIN_K", "2048"))


def rows_per_block(nrows_py, real_rows=None):
    """Rows per block as (Python expression of the sizes, C expression of
    RS_NROWS).

    One lane folds one row and a block is one warp, so the rows are dealt
    out as evenly as the SMs allow: R = ceil(rows / (2 x 148)) clamped to
    [MIN_ROWS, 32] gives two blocks on (nearly) every SM — 4096 rows -> 14,
    1024 (a strong-scaled band at 8 GPUs) -> 4 — except that a matrix of
    >= 8192 real rows (`real_rows`: (python, C) expressions; not the virtual
    rows of split rows) takes 32-row blocks: 256 blocks for 8192 rows
    measured 0.999-1.004 of the copy peak against 0.986-0.990 for the even
    28-row deal (293 blocks; profiles/gemv_rows_r02c.txt), while the split
    bands keep the even deal (32-row blocks: 2-3 % slower there)."""
    if ROWS:
        return str(ROWS), str(ROWS)
    slots = 2 * SM_COUNT
    lo = MIN_ROWS
    py = f"(32 if ({nrows_py}) > {32 * slots} else ({lo} if ({nrows_py}) <= {lo * slots} else -(-({nrows_py}) // {slots})))"
    c = f"(RS_NROWS > {32 * slots} ? 32 : RS_NROWS <= {lo * slots} ? {lo} : (RS_NROWS + {slots - 1}) / {slots})"
    if real_rows is not None:
        rpy, rc = real_rows
        py = f"(32 if ({rpy}) >= {32 * 256} else {py})"
        c = f"(({rc}) >= {32 * 256} ? 32 : {c})"
    return py, c


def affine_in_flat_row(base, loops, assumptions):
    """(c0, pitch, preconditions) with base == c0 + f * pitch for the flat row
    index f of the collapsed loops, or None."""
    row_vars = [v for v, _ in loops]
    zero = {v: nat.Const(0) for v in row_vars}
    c0 = nat.normalize(nat.substitute(base, zero), assumptions)
    coeffs = []
    for v in row_vars:
        one = dict(zero)
        one[v] = nat.Const(1)
        two = dict(zero)
        two[v] = nat.Const(2)
        c1 = nat.normalize(nat.substitute(base, one) - c0, assumptions)
        c2 = nat.normalize(nat.substitute(base, two) - c0, assumptions)
        if not nat.equal(c2, nat.normalize(c1 * nat.Const(2)), assumptions):
            return None
        if any(x in nat.free_vars(c1) for x in row_vars):
            return None
        coeffs.append(c1)
    pitch = coeffs[-1]
    pre = []
    inner = nat.Const(1)
    for k in range(len(loops) - 1, -1, -1):
        want = nat.normalize(pitch * inner, assumptions)
        if not nat.equal(coeffs[k], want, assumptions):
            pre.append(f"({py_expr(coeffs[k])}) == ({py_expr(want)})")
        inner = inner * loops[k][1]
    return c0, pitch, pre


def _is_sum_step(step, acc):
    """step == acc + e (or e + acc) with e free of acc, in fp32"""
    if not (isinstance(step, lir.Bin) and step.op == "+" and step.ctype == "float"):
        return False
    other = step.b if step.a == acc else step.a if step.b == acc else None
    return other is not None and acc not in set(lir.expr_scalars(other))


def emit(prog, loops, shape, row_streams, shared_streams, name, temps, exact, j_coef):
    """Render the kernel; returns (text, plan) or None if a precondition
    cannot be expressed."""
    acc, init, loop, post = shape
    step = loop.body.value
    r = NatRenderer(prog.clamps)
    nrows = nat.Const(1)
    for _, b in loops:
        nrows = nrows * b
    nrows = nat.normalize(nrows, prog.assumptions)
    n_py, k_py = py_expr(nrows), py_expr(loop.bound)

    rs_list = list(dict.fromkeys(row_streams.values()))
    sh_list = list(dict.fromkeys(shared_streams.values()))
    affs = []
    for buf, base in rs_list:
        aff = affine_in_flat_row(base, loops, prog.assumptions)
        if aff is None:
            return None
        affs.append(aff)
    split = SPLIT_TARGET > 0 and getattr(prog, "reassociate", False) and _is_sum_step(step, acc)
    if split:
        # S (a power of two <= 32) from the sizes, the same in Python (plan) and C
        conds_py = [f"({n_py}) < {SPLIT_TARGET}", f"({k_py}) >= {SPLIT_MIN_K}", f"({k_py}) % 128 == 0"]
        conds_c = [f"({r(nrows)}) < {SPLIT_TARGET}", f"({r(loop.bound)}) >= {SPLIT_MIN_K}", f"({r(loop.bound)}) % 128 == 0"]
        for _c0, pitch, _pre in affs:  # the chunks of a row are the rows of a [rows * S][K / S] view
            conds_py.append(f"({py_expr(pitch)}) == ({k_py})")
            conds_c.append(f"({r(pitch)}) == ({r(loop.bound)})")
        s_py = "(1 if not (" + " and ".join(conds_py) + ") else "
        s_c = "(!(" + " && ".join(conds_c) + ") ? 1 : "
        for sv in (2, 4, 8, 16):
            s_py += f"{sv} if ({n_py}) * {sv} >= {SPLIT_TARGET} else "
            s_c += f"({r(nrows)}) * {sv} >= {SPLIT_TARGET} ? {sv} : "
        s_py += "32)"
        s_c += "32)"
    else:
        s_py = s_c = "1"
    nv_py = f"(({n_py}) * {s_py})" if split else n_py
    kv_py = f"(({k_py}) // {s_py})" if split else k_py
    rows_py, rows_c = rows_per_block(nv_py, (n_py, r(nrows)))
    if split:  # a row's S chunks stay in one warp, S-aligned
        rows_py = f"(-(-({rows_py}) // {s_py}) * {s_py})"
        rows_c = f"((({rows_c}) + RS_S - 1) / RS_S * RS_S)"
    xs = KT + 4 if split else KT  # shared-stream segment stride (padded: S segments, conflict-free)

    # TMA boxes need non-empty tensors; 16-byte bulk copies need K % 4 == 0
    pre = [f"({k_py}) % 4 == 0", f"({k_py}) > 0", f"({n_py}) > 0"]
    tmaps = []
    for (buf, base), (c0, pitch, apre) in zip(rs_list, affs):
        pre += apre + [f"({py_expr(c0)}) % 4 == 0", f"({py_expr(pitch)}) % 4 == 0", f"({py_expr(pitch)}) > 0"]
        pitch_py = f"(({py_expr(pitch)}) // {s_py})" if split else py_expr(pitch)
        tmaps.append({"kind": "tma2d", "buf": buf, "offset": py_expr(c0), "dims": [kv_py, nv_py],
                      "pitch": pitch_py, "box": [32, rows_py], "swizzle": 3})
    for buf, base in sh_list:
        pre.append(f"({py_expr(base)}) % 4 == 0")
    pre = list(dict.fromkeys(pre))

    nbox = KT // 32
    # stages stay 1024-byte aligned (128B swizzle)
    boxrows_py = f"(-(-({rows_py}) // 8) * 8)"
    sh_py = f"{len(sh_list) * xs} * {s_py}" if split else f"{len(sh_list) * KT}"
    stage_py = f"(-(-({len(rs_list) * nbox * 32} * {boxrows_py} + {sh_py}) // 256) * 256)"
    # one stage (+ the 1024-byte alignment slack and the barriers) must fit the
    # 227 KiB opt-in shared memory; wider programs take the generic kernel
    pre.append(f"{stage_py} * 4 + 1024 + 64 <= 227 * 1024")
    # ring depth: up to STAGES (auto: MAX_STAGES), as many as the block's
    # budget holds — half the SM's shared memory when there are two blocks
    # per SM, all of it when the blocks fit one per SM (at least one stage:
    # a one-stage ring issues each stage just before it waits on it)
    cap = STAGES or MAX_STAGES
    nblk_py = f"(-(-({nv_py}) // {rows_py}))"
    budget_py = f"({220 * 1024} if {nblk_py} <= {SM_COUNT} else {113 * 1024})"
    stages_py = (f"({cap} if {budget_py} // ({stage_py} * 4) >= {cap} else "
                 f"(1 if {budget_py} // ({stage_py} * 4) < 1 else {budget_py} // ({stage_py} * 4)))")
    extra = [f"const __grid_constant__ rs_tmap rs_map{k}" for k in range(len(rs_list))]
    peer_out = int(getattr(prog, "peer_out", 0) or 0)
    if peer_out:
        # multi-GPU row bands with the result all-gathered INSIDE the kernel:
        # every row's value is also stored into every rank's full-result buffer
        # (peer memory over NVLink), then the ranks meet once per launch in
        # epoch-tagged slots (the dot exchange's protocol)
        if any(t.buf != prog.output.name for s_ in post for t, _v in lir.stmt_exprs(s_) if isinstance(t, lir.Store)):
            return None
        extra += ["const unsigned long long* __restrict__ rs_ytab", "const unsigned long long* __restrict__ rs_xtab",
                  "unsigned long long* __restrict__ rs_ticket"]
    lines = kernel_head(prog, name, temps, launch_bounds=32, extra_params=extra)
    if split:
        lines += [
            f"  // a row = RS_S contiguous column chunks folded by RS_S adjacent lanes (virtual rows of K / RS_S)",
            f"  constexpr int RS_S = {s_c}, RS_XS = {xs};",
            f"  constexpr int RS_NROWS = {r(nrows)} * RS_S;",
            f"  constexpr int RS_K = {r(loop.bound)} / RS_S;",
        ]
    else:
        lines += [
            f"  constexpr int RS_NROWS = {r(nrows)};",
            f"  constexpr int RS_K = {r(loop.bound)};",
        ]
    sh_c = f"{len(sh_list)} * RS_S * RS_XS" if split else f"{len(sh_list) * KT}"
    lines += [
        f"  constexpr int RS_ROWS = {rows_c}, RS_KT = {KT}, RS_NBOX = {nbox};",
        "  constexpr unsigned RS_MASK = RS_ROWS == 32 ? 0xffffffffu : (1u << RS_ROWS) - 1u;",
        "  constexpr int RS_BR = (RS_ROWS + 7) / 8 * 8;  // a box's rows in shared memory (1024-byte swizzle atoms)",
        "  constexpr int RS_NT = (RS_K + RS_KT - 1) / RS_KT;",
        f"  constexpr int RS_STAGE_FLOATS = ({len(rs_list) * nbox * 32} * RS_BR + {sh_c} + 255) / 256 * 256;",
        "  constexpr int RS_NBLK = (RS_NROWS + RS_ROWS - 1) / RS_ROWS;",
        f"  constexpr int RS_BUDGET = RS_NBLK <= {SM_COUNT} ? {220 * 1024} : {113 * 1024};  // one / two blocks per SM",
        "  constexpr int RS_FIT = RS_BUDGET / (RS_STAGE_FLOATS * 4);  // stages the block's budget holds",
        f"  constexpr int RS_STAGES = RS_FIT >= {cap} ? {cap} : (RS_FIT < 1 ? 1 : RS_FIT);",
        "  extern __shared__ __align__(1024) unsigned char rs_smem_raw[];",
        "  float* rs_smem = reinterpret_cast<float*>(rs_smem_raw + ((1024u - (rs_smem_addr(rs_smem_raw) & 1023u)) & 1023u));",
        "  unsigned long long* rs_bar = reinterpret_cast<unsigned long long*>(rs_smem + RS_STAGES * RS_STAGE_FLOATS);",
        "  const int rs_lane = threadIdx.x;  // the block is RS_ROWS lanes of one warp",
        "  const int rs_row0 = blockIdx.x * RS_ROWS;",
        "  const bool rs_active = rs_row0 + rs_lane < RS_NROWS;",
        "  const int rs_f = rs_active ? rs_row0 + rs_lane : RS_NROWS - 1;",
    ]
    if split:
        lines[-1] = "  const int rs_f = (rs_active ? rs_row0 + rs_lane : RS_NROWS - 1) / RS_S;  // the real row"
        lines.append("  const int rs_xo = (rs_lane % RS_S) * RS_XS;  // this lane's chunk of the shared streams")
    rest = "rs_f"
    for k, (var, _b) in enumerate(loops):
        if k == len(loops) - 1:
            lines.append(f"  const int {var} = {rest};")
        else:
            inner = nat.Const(1)
            for _, b in loops[k + 1:]:
                inner = inner * b
            size_c = r(nat.normalize(inner), 2)
            lines.append(f"  const int {var} = {rest} / {size_c};")
            lines.append(f"  const int rs_q{k} = {rest} % {size_c};")
            rest = f"rs_q{k}"
    for k, (buf, base) in enumerate(sh_list):
        lines.append(f"  const float* rs_gx{k} = {buf} + ({r(base)});")
    # per-lane swizzled chunk offsets (bytes) inside a 128-byte box row
    lines += [
        "  const int rs_sw = rs_lane & 7;",
        "  if (rs_lane == 0) {",
    ]
    for k in range(len(rs_list)):
        lines.append(f"    rs_tmap_prefetch(&rs_map{k});")
    lines += [
        "    for (int rs_s = 0; rs_s < RS_STAGES; ++rs_s) rs_mbar_init(&rs_bar[rs_s], 1);",
        "    rs_fence_barrier_init();",
        "  }",
        "  __syncwarp(RS_MASK);",
        "  auto rs_issue = [&](int rs_t) {",
        "    const int rs_slot = rs_t % RS_STAGES;",
        "    const int rs_j0 = rs_t * RS_KT;",
        "    const int rs_kt = RS_K - rs_j0 < RS_KT ? RS_K - rs_j0 : RS_KT;",
        "    const int rs_nb = (rs_kt + 31) / 32;",
        "    float* rs_st = rs_smem + rs_slot * RS_STAGE_FLOATS;",
        "    rs_fence_proxy_async();",
        "    if (rs_lane == 0) {",
        f"      rs_mbar_arrive_expect_tx(&rs_bar[rs_slot], (unsigned)(rs_nb * 128 * RS_ROWS * {len(rs_list)}"
        f" + rs_kt * 4 * {len(sh_list)}{' * RS_S' if split else ''}));",
    ]
    for k in range(len(rs_list)):
        lines += [
            "      for (int rs_b = 0; rs_b < rs_nb; ++rs_b)",
            f"        rs_tma_load_2d(rs_st + ({k} * RS_NBOX + rs_b) * 32 * RS_BR, &rs_map{k}, rs_j0 + 32 * rs_b, rs_row0,"
            " &rs_bar[rs_slot]);",
        ]
    for k in range(len(sh_list)):
        if split:
            off = f"{len(rs_list)} * RS_NBOX * 32 * RS_BR + {k} * RS_S * RS_XS"
            lines += [
                "      for (int rs_c = 0; rs_c < RS_S; ++rs_c)  // chunk c of the shared stream",
                f"        rs_bulk_g2s(rs_st + {off} + rs_c * RS_XS, rs_gx{k} + rs_c * RS_K + rs_j0, (unsigned)rs_kt * 4u,"
                " &rs_bar[rs_slot]);",
            ]
        else:
            off = f"{len(rs_list)} * RS_NBOX * 32 * RS_BR + {k} * RS_KT"
            lines.append(f"      rs_bulk_g2s(rs_st + {off}, rs_gx{k} + rs_j0, (unsigned)rs_kt * 4u, &rs_bar[rs_slot]);")
    lines += [
        "    }",
        "  };",
        "  for (int rs_t = 0; rs_t < RS_STAGES - 1 && rs_t < RS_NT; ++rs_t) rs_issue(rs_t);",
    ]
    vr = ValueRenderer(prog, exact)
    lines.append(f"  {acc.ctype} {acc.name};")
    if split:  # chunks after the first start from the identity of the sum
        lines.append(f"  {acc.name} = rs_lane % RS_S == 0 ? ({vr(init.value)}) : ({acc.ctype})0;")
    else:
        lines.append(f"  {acc.name} = {vr(init.value)};")
    xoff = " + rs_xo" if split else ""
    xstride = "RS_S * RS_XS" if split else "RS_KT"

    def step_with(comp):
        def hook(ld):
            if ld in row_streams:
                return f"rs_a{rs_list.index(row_streams[ld])}.{comp}"
            if ld in shared_streams:
                return f"rs_x{sh_list.index(shared_streams[ld])}.{comp}"
            return None

        return ValueRenderer(prog, exact, load_hook=hook)(step)

    def chunk(ind):
        p = " " * ind
        out = [
            f"{p}const int rs_box = rs_jj >> 5;",
            f"{p}const int rs_chunk = ((rs_jj >> 2) & 7) ^ rs_sw;",
        ]
        for k in range(len(rs_list)):
            out.append(
                f"{p}const float4 rs_a{k} = *reinterpret_cast<const float4*>(rs_st + ({k} * RS_NBOX + rs_box) * 32 * RS_BR"
                f" + rs_lane * 32 + rs_chunk * 4);")
        for k in range(len(sh_list)):
            off = f"{len(rs_list)} * RS_NBOX * 32 * RS_BR + {k} * {xstride}{xoff}"
            out.append(f"{p}const float4 rs_x{k} = *reinterpret_cast<const float4*>(rs_st + {off} + rs_jj);")
        for comp in ("x", "y", "z", "w"):
            out.append(f"{p}{acc.name} = {step_with(comp)};")
        return out

    def chunk_pf(ind):
        """A full stage's fold with the shared-memory reads PF chunks ahead
        of their use (a register ring): the fold is one dependent add per
        column, so with one warp per SM sub-partition an LDS issued just
        before its use (~30 cycles) would stall every chunk."""
        p = " " * ind
        names = [f"rs_a{k}" for k in range(len(rs_list))] + [f"rs_x{k}" for k in range(len(sh_list))]

        def loads(slot, jj):
            out = [
                f"{p}  const int rs_box = ({jj}) >> 5;",
                f"{p}  const int rs_chunk = ((({jj}) >> 2) & 7) ^ rs_sw;",
            ]
            for k in range(len(rs_list)):
                out.append(f"{p}  rs_pa{k}[{slot}] = *reinterpret_cast<const float4*>(rs_st + ({k} * RS_NBOX + rs_box)"
                           " * 32 * RS_BR + rs_lane * 32 + rs_chunk * 4);")
            for k in range(len(sh_list)):
                off = f"{len(rs_list)} * RS_NBOX * 32 * RS_BR + {k} * {xstride}{xoff}"
                out.append(f"{p}  rs_px{k}[{slot}] = *reinterpret_cast<const float4*>(rs_st + {off} + ({jj}));")
            return out

        out = [f"{p}float4 " + ", ".join(f"rs_p{n[3]}{n[4:]}[{PF}]" for n in names) + ";"]
        out += [f"{p}#pragma unroll", f"{p}for (int rs_d = 0; rs_d < {PF}; ++rs_d) {{"]
        out += loads("rs_d", "4 * rs_d")
        out += [f"{p}}}", f"{p}#pragma unroll", f"{p}for (int rs_jj = 0; rs_jj < RS_KT; rs_jj += 4) {{",
                f"{p}  const int rs_c = (rs_jj >> 2) % {PF};"]
        out += [f"{p}  const float4 {n} = rs_p{n[3]}{n[4:]}[rs_c];" for n in names]
        out += [f"{p}  if (rs_jj + {4 * PF} < RS_KT) {{"]
        out += ["  " + x for x in loads("rs_c", f"rs_jj + {4 * PF}")]
        out += [f"{p}  }}"]
        for comp in ("x", "y", "z", "w"):
            out.append(f"{p}  {acc.name} = {step_with(comp)};")
        out += [f"{p}}}"]
        return out

    lines += [
        "  for (int rs_t = 0; rs_t < RS_NT; ++rs_t) {",
        "    if (rs_t + RS_STAGES - 1 < RS_NT) rs_issue(rs_t + RS_STAGES - 1);",
        "    const int rs_slot = rs_t % RS_STAGES;",
        "    const float* rs_st = rs_smem + rs_slot * RS_STAGE_FLOATS;",
        "    rs_mbar_wait(&rs_bar[rs_slot], (unsigned)((rs_t / RS_STAGES) & 1));",
        "    const int rs_kt = RS_K - rs_t * RS_KT < RS_KT ? RS_K - rs_t * RS_KT : RS_KT;",
        "    if (rs_kt == RS_KT) {",
    ]
    if PF:
        lines += chunk_pf(6)
    else:
        lines += ["#pragma unroll", "      for (int rs_jj = 0; rs_jj < RS_KT; rs_jj += 4) {"]
        lines += chunk(8)
        lines += ["      }"]
    lines += [
        "    } else {",
        "      for (int rs_jj = 0; rs_jj < rs_kt; rs_jj += 4) {",
    ]
    lines += chunk(8)
    lines += [
        "      }",
        "    }",
        "    __syncwarp(RS_MASK);",
        "  }",
    ]
    if split:
        add = "__fadd_rn" if (exact and acc.ctype == "float") else ""
        lines += [
            "  if (RS_S > 1) {",
            "    // the RS_S chunk partials of a row sit in RS_S adjacent lanes: the first adds",
            "    // the others to its own in chunk order",
            "    const int rs_g = rs_lane & ~(RS_S - 1);",
            f"    {acc.ctype} rs_tot = {acc.name};",
            "#pragma unroll",
            "    for (int rs_c = 1; rs_c < RS_S; ++rs_c)",
            (f"      rs_tot = {add}(rs_tot, __shfl_sync(RS_MASK, {acc.name}, rs_g + rs_c));" if add else
             f"      rs_tot = rs_tot + __shfl_sync(RS_MASK, {acc.name}, rs_g + rs_c);"),
            f"    {acc.name} = rs_tot;",
            "  }",
            "  if (rs_active && rs_lane % RS_S == 0) {",
        ]
    else:
        lines.append("  if (rs_active) {")
    from .emit_cuda import GenericKernel, Stage

    for s in post:
        g = GenericKernel(prog, Stage("serial", s), "_", [], exact)
        lines += [("    " + x) for x in g.thread(s, 0)]
    if peer_out:
        out_name = prog.output.name
        lines += [
            f"    // the same stores into every rank's full buffer, at this rank's row offset",
            f"    for (int rs_k = 0; rs_k < {peer_out}; ++rs_k) {{",
            f"      float* const {out_name} = reinterpret_cast<float*>(rs_ytab[rs_k]) + rs_ytab[{peer_out}];",
        ]
        for s_ in post:
            g = GenericKernel(prog, Stage("serial", s_), "_", [], exact)
            lines += [("      " + x) for x in g.thread(s_, 0)]
        lines += ["    }"]
    lines += ["  }"]
    if peer_out:
        lines += [
            "  // this block's peer stores are visible system-wide before its ticket; the",
            "  // launch's last block then publishes the epoch to every rank and waits for",
            "  // every rank's: when the kernel ends, every rank's full buffer is complete",
            "  __threadfence_system();",
            "  __syncwarp(RS_MASK);",
            "  if (rs_lane == 0) {",
            "    const unsigned long long rs_t = atomicAdd(rs_ticket, 1ull);",
            "    if (rs_t % gridDim.x == gridDim.x - 1) {",
            "      __threadfence_system();  // acquire side: every block's fenced stores precede the publish",
            "      const unsigned rs_e = (unsigned)(rs_t / gridDim.x) + 1u;",
            f"      constexpr int RS_R = {peer_out};",
            "      const int rs_me = (int)rs_xtab[RS_R];",
            "      const int rs_bank = (int)(rs_e & 1u) * RS_R;  // two banks by epoch parity (PeerExchange)",
            "      for (int rs_k = 0; rs_k < RS_R; ++rs_k)",
            "        rs_xchg_put(reinterpret_cast<unsigned long long*>(rs_xtab[rs_k]) + rs_bank + rs_me, rs_e, 1u);",
            "      const unsigned long long* rs_slots = reinterpret_cast<const unsigned long long*>(rs_xtab[rs_me]) + rs_bank;",
            "      for (int rs_k = 0; rs_k < RS_R; ++rs_k) (void)rs_xchg_get(rs_slots + rs_k, rs_e);",
            "    }",
            "  }",
        ]
    lines += ["}"]
    smem = f"{stages_py} * {stage_py} * 4 + {stages_py} * 8 + 1024"
    plan = {
        "name": name,
        "kind": "rowfold",
        "rows": py_expr(nrows),
        "row_block": rows_py,
        "smem": smem,
        "pre": pre,
        "fmad": False,
        "order": "preserved",
        "extra_args": tmaps,
    }
    if split:
        plan["rows"] = nv_py
        plan["split"] = s_py
        plan["order"] = (f"preserved when split == 1 (rows >= {SPLIT_TARGET}, K < {SPLIT_MIN_K} or strided rows); "
                         "else `split` contiguous column chunks per row, partials added in chunk order")
    if peer_out:
        ws_t = f"rs_ws_{name}_ticket"
        plan.update(peer_out=peer_out, workspace=[{"name": ws_t, "ctype": "int", "size": "2"}])
        plan["extra_args"] = tmaps + [{"kind": "peer_ptr_table", "name": "rs_y_table"},
                                      {"kind": "peer_table"}, {"kind": "workspace", "name": ws_t}]
    return "\n".join(lines) + "\n", plan
