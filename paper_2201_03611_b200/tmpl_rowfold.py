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
STAGES = int(os.environ.get("RISE_ROWFOLD_STAGES", "3"))
SM_COUNT = 148


def rows_per_block(nrows_py):
    """Rows per block as (Python expression of the sizes, C expression of
    RS_NROWS).

    One lane folds one row and a block is one warp, so the rows are dealt
    out as evenly as the SMs allow: R = ceil(rows / (2 x 148)) clamped to
    [8, 32] gives two blocks on (nearly) every SM.  8192 rows -> 28 rows
    per block, 293 blocks (with 32 rows, 256 blocks leave 40 SMs one block
    and 108 two: the two-block SMs set the time); 4096 rows -> 14."""
    if ROWS:
        return str(ROWS), str(ROWS)
    slots = 2 * SM_COUNT
    return (f"(32 if ({nrows_py}) > {32 * slots} else (8 if ({nrows_py}) <= {8 * slots} else -(-({nrows_py}) // {slots})))",
            f"(RS_NROWS > {32 * slots} ? 32 : RS_NROWS <= {8 * slots} ? 8 : (RS_NROWS + {slots - 1}) / {slots})")


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
    rows_py, rows_c = rows_per_block(py_expr(nrows))

    rs_list = list(dict.fromkeys(row_streams.values()))
    sh_list = list(dict.fromkeys(shared_streams.values()))
    # TMA boxes need non-empty tensors; 16-byte bulk copies need K % 4 == 0
    pre = [f"({py_expr(loop.bound)}) % 4 == 0", f"({py_expr(loop.bound)}) > 0", f"({py_expr(nrows)}) > 0"]
    tmaps = []
    for k, (buf, base) in enumerate(rs_list):
        aff = affine_in_flat_row(base, loops, prog.assumptions)
        if aff is None:
            return None
        c0, pitch, apre = aff
        pre += apre + [f"({py_expr(c0)}) % 4 == 0", f"({py_expr(pitch)}) % 4 == 0", f"({py_expr(pitch)}) > 0"]
        tmaps.append({"kind": "tma2d", "buf": buf, "offset": py_expr(c0), "dims": [py_expr(loop.bound), py_expr(nrows)],
                      "pitch": py_expr(pitch), "box": [32, rows_py], "swizzle": 3})
    for buf, base in sh_list:
        pre.append(f"({py_expr(base)}) % 4 == 0")
    pre = list(dict.fromkeys(pre))

    nbox = KT // 32
    # stages stay 1024-byte aligned (128B swizzle)
    boxrows_py = f"(-(-({rows_py}) // 8) * 8)"
    stage_py = f"(-(-({len(rs_list) * nbox * 32} * {boxrows_py} + {len(sh_list) * KT}) // 256) * 256)"
    # one stage (+ the 1024-byte alignment slack and the barriers) must fit the
    # 227 KiB opt-in shared memory; wider programs take the generic kernel
    pre.append(f"{stage_py} * 4 + 1024 + 64 <= 227 * 1024")
    # ring depth: up to STAGES, as many as fit two blocks per SM for the block's rows
    # (at least one: a one-stage ring issues each stage just before it waits on it)
    budget = 113 * 1024
    stages_py = (f"({STAGES} if {budget} // ({stage_py} * 4) >= {STAGES} else "
                 f"(1 if {budget} // ({stage_py} * 4) < 1 else {budget} // ({stage_py} * 4)))")
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
    lines += [
        f"  constexpr int RS_NROWS = {r(nrows)};",
        f"  constexpr int RS_ROWS = {rows_c}, RS_KT = {KT}, RS_NBOX = {nbox};",
        "  constexpr unsigned RS_MASK = RS_ROWS == 32 ? 0xffffffffu : (1u << RS_ROWS) - 1u;",
        "  constexpr int RS_BR = (RS_ROWS + 7) / 8 * 8;  // a box's rows in shared memory (1024-byte swizzle atoms)",
        f"  constexpr int RS_K = {r(loop.bound)};",
        "  constexpr int RS_NT = (RS_K + RS_KT - 1) / RS_KT;",
        f"  constexpr int RS_STAGE_FLOATS = ({len(rs_list) * nbox * 32} * RS_BR + {len(sh_list) * KT} + 255) / 256 * 256;",
        f"  constexpr int RS_FIT = {budget} / (RS_STAGE_FLOATS * 4);  // stages two blocks per SM can hold",
        f"  constexpr int RS_STAGES = RS_FIT >= {STAGES} ? {STAGES} : (RS_FIT < 1 ? 1 : RS_FIT);",
        "  extern __shared__ __align__(1024) unsigned char rs_smem_raw[];",
        "  float* rs_smem = reinterpret_cast<float*>(rs_smem_raw + ((1024u - (rs_smem_addr(rs_smem_raw) & 1023u)) & 1023u));",
        "  unsigned long long* rs_bar = reinterpret_cast<unsigned long long*>(rs_smem + RS_STAGES * RS_STAGE_FLOATS);",
        "  const int rs_lane = threadIdx.x;  // the block is RS_ROWS lanes of one warp",
        "  const int rs_row0 = blockIdx.x * RS_ROWS;",
        "  const bool rs_active = rs_row0 + rs_lane < RS_NROWS;",
        "  const int rs_f = rs_active ? rs_row0 + rs_lane : RS_NROWS - 1;",
    ]
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
        f" + rs_kt * 4 * {len(sh_list)}));",
    ]
    for k in range(len(rs_list)):
        lines += [
            "      for (int rs_b = 0; rs_b < rs_nb; ++rs_b)",
            f"        rs_tma_load_2d(rs_st + ({k} * RS_NBOX + rs_b) * 32 * RS_BR, &rs_map{k}, rs_j0 + 32 * rs_b, rs_row0,"
            " &rs_bar[rs_slot]);",
        ]
    for k in range(len(sh_list)):
        off = f"{len(rs_list)} * RS_NBOX * 32 * RS_BR + {k} * RS_KT"
        lines.append(f"      rs_bulk_g2s(rs_st + {off}, rs_gx{k} + rs_j0, (unsigned)rs_kt * 4u, &rs_bar[rs_slot]);")
    lines += [
        "    }",
        "  };",
        "  for (int rs_t = 0; rs_t < RS_STAGES - 1 && rs_t < RS_NT; ++rs_t) rs_issue(rs_t);",
    ]
    vr = ValueRenderer(prog, exact)
    lines.append(f"  {acc.ctype} {acc.name};")
    lines.append(f"  {acc.name} = {vr(init.value)};")

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
            off = f"{len(rs_list)} * RS_NBOX * 32 * RS_BR + {k} * RS_KT"
            out.append(f"{p}const float4 rs_x{k} = *reinterpret_cast<const float4*>(rs_st + {off} + rs_jj);")
        for comp in ("x", "y", "z", "w"):
            out.append(f"{p}{acc.name} = {step_with(comp)};")
        return out

    lines += [
        "  for (int rs_t = 0; rs_t < RS_NT; ++rs_t) {",
        "    if (rs_t + RS_STAGES - 1 < RS_NT) rs_issue(rs_t + RS_STAGES - 1);",
        "    const int rs_slot = rs_t % RS_STAGES;",
        "    const float* rs_st = rs_smem + rs_slot * RS_STAGE_FLOATS;",
        "    rs_mbar_wait(&rs_bar[rs_slot], (unsigned)((rs_t / RS_STAGES) & 1));",
        "    const int rs_kt = RS_K - rs_t * RS_KT < RS_KT ? RS_K - rs_t * RS_KT : RS_KT;",
        "    if (rs_kt == RS_KT) {",
        "#pragma unroll",
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
        "    __syncwarp(RS_MASK);",
        "  }",
        "  if (rs_active) {",
    ]
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
    if peer_out:
        ws_t = f"rs_ws_{name}_ticket"
        plan.update(peer_out=peer_out, workspace=[{"name": ws_t, "ctype": "int", "size": "2"}])
        plan["extra_args"] = tmaps + [{"kind": "peer_ptr_table", "name": "rs_y_table"},
                                      {"kind": "peer_table"}, {"kind": "workspace", "name": ws_t}]
    return "\n".join(lines) + "\n", plan
