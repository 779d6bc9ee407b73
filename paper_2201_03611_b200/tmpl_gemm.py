"""`gemm_tc` template: the dense contraction on tcgen05 tensor cores (3xTF32).

Matches the sgemm program's loop nest (programs.SGEMM_BT, SURVEY.md §8 c):

    for i < M, j < N (parallel):
        acc = 0.0f
        for p < K:  acc = acc + A[i*K + p] * Bt[j*K + p]     (either product order)
        output[i*N + j] = acc

and instantiates rise/gemm_tc.cuh: TMA-fed, 128x128 CTA tiles, fp32
accumulation in tensor memory, operands split hi/lo in shared memory.

Order/precision: REASSOCIATED.  The tensor core sums K in its own order and
the operands pass through the 3xTF32 split, so parity is the fp64 error
bound |C - C64| <= 2 K u (|A||B|) of SURVEY.md §8 d, not bit equality.
"""

from __future__ import annotations

import os

from . import lir
from ._ref import nat
from .emit_cuda import NatRenderer, kernel_head, py_expr

# tile width, pipeline depth and whether the converter writes hi tiles back
# (overridable for tuning sweeps only)
BN = int(os.environ.get("RISE_GEMM_BN", "256"))
STAGES = int(os.environ.get("RISE_GEMM_STAGES", "2"))
WRITE_HI = os.environ.get("RISE_GEMM_WRITE_HI", "0") == "1"
# CTA-pair (cta_group::2, M = 256) variant
PAIR = os.environ.get("RISE_GEMM_2SM", "1") == "1"
PAIR_BN = int(os.environ.get("RISE_GEMM_PAIR_BN", "256"))
PAIR_STAGES = int(os.environ.get("RISE_GEMM_PAIR_STAGES", "3"))
# persistent CTA pairs with a double-buffered TMEM accumulator and dedicated
# epilogue warps (gemm_3xtf32_2sm_persistent)
GROUP_M = int(os.environ.get("RISE_GEMM_GROUP_M", "8"))  # persistent tile order: groups of 8 row tiles, column by column (measured +0.6 %; 0 = row-major)
PERSIST = os.environ.get("RISE_GEMM_PERSIST", "1") == "1"  # measured 278 -> 284 TFLOP/s


def match(prog, stage, base_name, temps, exact, parallel_rows, fold_shape):
    """The flat nest (programs.SGEMM_BT / SGEMM): two parallel loops over the
    output and one fold over K."""
    loops, body = parallel_rows(stage)
    if loops is None or len(loops) != 2 or stage.kind != "grid":
        return None
    (iv, M), (jv, N) = loops
    shape = fold_shape(body)
    if shape is None:
        return None
    acc, init, loop, post = shape
    if not _zero(init.value):
        return None
    step = _product_step(loop.body.value, acc)
    if step is None:
        return None
    if len(post) != 1:
        return None
    V = nat.Var
    desc = _operands(prog, step[0], step[1], V(iv), V(jv), V(loop.var), M, N, loop.bound, post[0])
    if desc is None or desc["value"] != acc:
        return None
    return emit(prog, desc, base_name, temps)


def _zero(value):
    return isinstance(value, lir.Lit) and value.text in ("0.0f", "0f", "0.0")


def _product_step(step, acc):
    """acc + x * y (fp32, two loads) -> (x, y)."""
    if not (isinstance(step, lir.Bin) and step.op == "+" and step.a == acc and isinstance(step.b, lir.Bin)
            and step.b.op == "*" and isinstance(step.b.a, lir.Load) and isinstance(step.b.b, lir.Load)
            and step.ctype == "float"):
        return None
    return step.b.a, step.b.b


def _operands(prog, x, y, I, J, P, M, N, K, store):
    """Which load is A[I][P] and which B (as Bt[J][P], K-major, or B[P][J],
    MN-major), with the result stored at output[I][J]; None otherwise."""

    def idx(ld):
        return ld.index

    def is_row(ld, row):
        return nat.equal(idx(ld), nat.normalize(row * K + P), prog.assumptions)

    def is_col(ld):  # B[k][j] of a row-major K x N matrix (e.g. read through transpose(B))
        return nat.equal(idx(ld), nat.normalize(P * N + J), prog.assumptions)

    b_mn = False  # B is MN-major in shared memory (UMMA b_major = 1)
    if is_row(x, I) and is_row(y, J):
        a_ld, b_ld = x, y
    elif is_row(y, I) and is_row(x, J):
        a_ld, b_ld = y, x
    elif PAIR and is_row(x, I) and is_col(y):
        a_ld, b_ld, b_mn = x, y, True
    elif PAIR and is_row(y, I) and is_col(x):
        a_ld, b_ld, b_mn = y, x, True
    else:
        return None
    for ld in (a_ld, b_ld):
        if prog.buffers[ld.buf].role != "input" or ld.ctype != "float":
            return None
    if not (isinstance(store, lir.Assign) and isinstance(store.target, lir.Store)
            and nat.equal(store.target.index, nat.normalize(I * N + J), prog.assumptions)):
        return None
    return {"M": M, "N": N, "K": K, "a": a_ld.buf, "b": b_ld.buf, "b_mn": b_mn, "out": store.target.buf,
            "value": store.value}


# ---------------------------------------------------------------------------
# the tiled nest (programs.SGEMM_TILED): workgroups over row blocks of A, the
# block staged in Local memory, work-items over the columns, K in tiles


def _copy_nest(stmt):
    """(Par)For nest ending in L[dst] = S[src] (or S[src] * 1.0f): returns
    (L, S, dst, src, [(var, bound)]) or None."""
    loops = []
    while isinstance(stmt, (lir.For, lir.ParFor)):
        if isinstance(stmt, lir.ParFor) and stmt.kind != "local":
            return None
        loops.append((stmt.var, stmt.bound))
        stmt = stmt.body
    if not (isinstance(stmt, lir.Assign) and isinstance(stmt.target, lir.Store)):
        return None
    v = stmt.value
    if isinstance(v, lir.Bin) and v.op == "*":
        if isinstance(v.b, lir.Lit) and v.b.text == "1.0f":
            v = v.a
        elif isinstance(v.a, lir.Lit) and v.a.text == "1.0f":
            v = v.b
    if not isinstance(v, lir.Load):
        return None
    return stmt.target.buf, v.buf, stmt.target.index, v.index, loops


def _staged(prog, stmt, allocs):
    """Peel Local staging buffers: Alloc(L, Local){ Seq[copy into L, rest] }.
    Returns (compute statement, {L: (source buffer, offset Nat)}) or None."""
    stage_map = {}
    while True:
        if isinstance(stmt, lir.Alloc) and stmt.space == "Local" and stmt.dims:
            allocs[stmt.name] = stmt
            stmt = stmt.body
            continue
        if isinstance(stmt, lir.Seq) and len(stmt.stmts) >= 2:
            info = _copy_nest(stmt.stmts[0])
            if info is None or info[0] not in allocs:
                return None
            L, src, dst, sidx, loops = info
            # the copy visits every element of L once, in row-major order ...
            size = nat.Const(1)
            expect = nat.Const(0)
            for var, bound in loops:
                expect = expect * bound + nat.Var(var)
                size = size * bound
            dims = allocs[L].dims
            total = nat.Const(1)
            for d in dims:
                total = total * d
            if not (nat.equal(nat.normalize(dst), nat.normalize(expect), prog.assumptions)
                    and nat.equal(nat.normalize(size), nat.normalize(total), prog.assumptions)):
                return None
            # ... from a contiguous run of the source: L[e] == S[e + delta]
            delta = nat.normalize(sidx - dst, prog.assumptions)
            if nat.free_vars(delta) & {v for v, _ in loops}:
                return None
            if prog.buffers[src].role != "input" or src in stage_map:
                return None
            stage_map[L] = (src, delta)
            rest = stmt.stmts[1:]
            stmt = rest[0] if len(rest) == 1 else lir.Seq(list(rest))
            continue
        return stmt, stage_map


def _through_staging(ld, stage_map, assumptions):
    if ld.buf in stage_map:
        src, delta = stage_map[ld.buf]
        return lir.Load(src, nat.normalize(ld.index + delta, assumptions), ld.ctype)
    return ld


def _k_fold(prog, body, fold_shape):
    """The per-output fold: either acc = 0; for p < K: acc += x*y; store — or
    K in tiles: P[t] = (fold over kk < TK of x*y) for t < T, then
    acc = 0; for t < T: acc += P[t]; store.  Returns (x, y, P expr, K, store,
    the stored accumulator)."""
    shape = fold_shape(body)
    if shape is not None:
        acc, init, loop, post = shape
        step = _product_step(loop.body.value, acc)
        if not _zero(init.value) or step is None or len(post) != 1:
            return None
        return step[0], step[1], nat.Var(loop.var), loop.bound, post[0], acc
    if not (isinstance(body, lir.Alloc) and body.space == "Private" and len(body.dims) == 1):
        return None
    parts = body.name
    T = body.dims[0]
    stmts = body.body.stmts if isinstance(body.body, lir.Seq) else [body.body]
    if len(stmts) != 2 or not isinstance(stmts[0], lir.For) or not nat.equal(stmts[0].bound, T, prog.assumptions):
        return None
    t = stmts[0].var
    inner = fold_shape(stmts[0].body)
    if inner is None:
        return None
    acc, init, loop, post = inner
    step = _product_step(loop.body.value, acc)
    if not _zero(init.value) or step is None or len(post) != 1:
        return None
    p0 = post[0]
    if not (isinstance(p0, lir.Assign) and isinstance(p0.target, lir.Store) and p0.target.buf == parts
            and nat.equal(p0.target.index, nat.Var(t)) and p0.value == acc):
        return None
    outer = fold_shape(stmts[1])
    if outer is None:
        return None
    acc2, init2, loop2, post2 = outer
    v = loop2.body.value
    if not (_zero(init2.value) and isinstance(v, lir.Bin) and v.op == "+" and v.a == acc2
            and isinstance(v.b, lir.Load) and v.b.buf == parts and nat.equal(v.b.index, nat.Var(loop2.var))
            and nat.equal(loop2.bound, T, prog.assumptions) and len(post2) == 1):
        return None
    TK = loop.bound
    P = nat.normalize(TK * nat.Var(t) + nat.Var(loop.var))
    return step[0], step[1], P, nat.normalize(T * TK, prog.assumptions), post2[0], acc2


def match_tiled(prog, stage, base_name, temps, exact, fold_shape):
    if stage.kind != "workgroup" or not PAIR:
        return None
    wg = stage.stmt
    got = _staged(prog, wg.body, {})
    if got is None:
        return None
    compute, stage_map = got
    chain = []
    s = compute
    while isinstance(s, (lir.For, lir.ParFor)) and len(chain) < 2:
        if isinstance(s, lir.ParFor) and s.kind != "local":
            return None
        chain.append(s)
        s = s.body
    if len(chain) != 2 or not any(isinstance(c, lir.ParFor) for c in chain):
        return None
    fold = _k_fold(prog, s, fold_shape)
    if fold is None:
        return None
    x, y, P, K, store, _acc = fold
    x = _through_staging(x, stage_map, prog.assumptions)
    y = _through_staging(y, stage_map, prog.assumptions)
    V = nat.Var
    for row, col in ((chain[0], chain[1]), (chain[1], chain[0])):
        TM = row.bound
        if not isinstance(TM, nat.Const):
            continue
        I = nat.normalize(TM * V(wg.var) + V(row.var))
        M = nat.normalize(wg.bound * TM, prog.assumptions)
        desc = _operands(prog, x, y, I, V(col.var), P, M, col.bound, K, store)
        if desc is not None and desc["value"] == fold[5]:
            return emit(prog, desc, base_name, temps)
    return None


def emit(prog, desc, base_name, temps):
    """The gemm_tc kernel and plan for C[M x N] = A[M x K] * B (desc)."""
    M, N, K = desc["M"], desc["N"], desc["K"]
    b_mn = desc["b_mn"]
    a_buf, b_buf, out_buf = desc["a"], desc["b"], desc["out"]
    name = f"{base_name}_gemm"
    r = NatRenderer(prog.clamps)
    bn, stages, write_hi = BN, STAGES, WRITE_HI
    extra = ["const __grid_constant__ rs_tmap rs_mapA", "const __grid_constant__ rs_tmap rs_mapB"]
    if PAIR:
        extra += ["int rs_nfull", "float* __restrict__ rs_ws", "unsigned* __restrict__ rs_flags"]
        if PERSIST:
            extra[3:3] = ["int rs_nunits", "int rs_ksplit"]
    threads = 320 if (PAIR and PERSIST) else 192
    lines = kernel_head(prog, name, temps, launch_bounds=f"{threads}, 1", extra_params=extra)
    if PAIR:
        fn = "gemm_3xtf32_2sm_persistent" if PERSIST else "gemm_3xtf32_2sm"
        args = "rs_nfull, rs_nunits, rs_ksplit, rs_ws, rs_flags" if PERSIST else "rs_nfull, rs_ws, rs_flags"
        lines += [
            f"  rise_gemm::{fn}<{r(M)}, {r(N)}, {r(K)}, {PAIR_BN}, {PAIR_STAGES}, "
            f"{'true' if b_mn else 'false'}{(', ' + str(GROUP_M)) if PERSIST and GROUP_M else ''}>"
            f"({out_buf}, {r(N)}, &rs_mapA, &rs_mapB, {args});",
            "}",
        ]
        plan = {
            "name": name,
            "kind": "gemm_tc",
            "M": py_expr(M),
            "N": py_expr(N),
            "K": py_expr(K),
            "bn": PAIR_BN,
            "pair": True,
            "b_major": "mn" if b_mn else "k",
            "persistent": PERSIST,
            "fmad": False,
            "order": ("3xtf32 tensor-core, CTA pairs; tail tiles K-split in two halves, or every tile in up to 4 "
                      "K ranges when there are fewer tiles than SM pairs (reassociated)"),
            # ragged M / N / K: TMA zero-fill + a guarded epilogue; the 16-byte
            # row pitch of the TMA views needs K % 4 (and N % 4 for MN-major B)
            "pre": [f"({py_expr(K)}) % 4 == 0", f"({py_expr(M)}) * ({py_expr(N)}) * ({py_expr(K)}) > 0"]
                   + ([f"({py_expr(N)}) % 4 == 0"] if b_mn else []),
            "smem": PAIR_STAGES * 2 * (128 * 32 * 4 + (PAIR_BN // 2) * 32 * 4) + 1024 + 256,
            "extra_args": [
                {"kind": "tma2d", "buf": a_buf, "offset": "0", "dims": [py_expr(K), py_expr(M)],
                 "pitch": py_expr(K), "box": [32, 128], "swizzle": 3},
                ({"kind": "tma2d", "buf": b_buf, "offset": "0", "dims": [py_expr(N), py_expr(K)],
                  "pitch": py_expr(N), "box": [32, 32], "swizzle": 4} if b_mn else
                 {"kind": "tma2d", "buf": b_buf, "offset": "0", "dims": [py_expr(K), py_expr(N)],
                  "pitch": py_expr(K), "box": [32, PAIR_BN // 2], "swizzle": 3}),
                {"kind": "gemm_full_tiles", "M": py_expr(M), "N": py_expr(N), "K": py_expr(K), "bn": PAIR_BN},
                *([{"kind": "gemm_units", "M": py_expr(M), "N": py_expr(N), "K": py_expr(K), "bn": PAIR_BN},
                   {"kind": "gemm_ksplit", "M": py_expr(M), "N": py_expr(N), "K": py_expr(K), "bn": PAIR_BN}]
                  if PERSIST else []),
                {"kind": "workspace", "name": f"rs_ws_{base_name}_ktail"},
                {"kind": "workspace", "name": f"rs_ws_{base_name}_kflags"},
            ],
            # K-split tiles park their parts 1.. here: (parts - 1) x split tiles <= one wave of pair tiles
            "workspace": [{"name": f"rs_ws_{base_name}_ktail", "ctype": "float", "size": f"74 * 256 * {PAIR_BN}"},
                          {"name": f"rs_ws_{base_name}_kflags", "ctype": "int", "size": "4 * 74"}],
        }
        return "\n".join(lines) + "\n", plan
    lines += [
        f"  rise_gemm::gemm_3xtf32<{r(K)}, {bn}, {stages}, {'true' if write_hi else 'false'}>"
        f"({out_buf}, {r(N)}, &rs_mapA, &rs_mapB);",
        "}",
    ]
    plan = {
        "name": name,
        "kind": "gemm_tc",
        "M": py_expr(M),
        "N": py_expr(N),
        "bn": bn,
        "fmad": False,
        "order": "3xtf32 tensor-core (reassociated)",
        "pre": [f"({py_expr(M)}) % 128 == 0", f"({py_expr(N)}) % {bn} == 0", f"({py_expr(K)}) % 32 == 0",
                f"({py_expr(M)}) * ({py_expr(N)}) * ({py_expr(K)}) > 0"],
        "smem": stages * 2 * (128 * 32 * 4 + bn * 32 * 4) + 1024 + 256,
        "extra_args": [
            {"kind": "tma2d", "buf": a_buf, "offset": "0", "dims": [py_expr(K), py_expr(M)], "pitch": py_expr(K),
             "box": [32, 128], "swizzle": 3},
            {"kind": "tma2d", "buf": b_buf, "offset": "0", "dims": [py_expr(K), py_expr(N)], "pitch": py_expr(K),
             "box": [32, bn], "swizzle": 3},
        ],
    }
    return "\n".join(lines) + "\n", plan


SPLIT_SLOTS_MAX = 74  # workspace sizing: at most this many split tiles (one wave of B200 SM pairs)


def pair_tiles(M, N, bn):
    return -(-M // 256) * -(-N // bn)


def schedule(M, N, K, bn, sm, persistent=PERSIST):
    """(whole tiles, K parts per split tile).  Whole tiles run first; the rest
    are split along K so the last wave fills the SM pairs:
      * at least a wave of tiles: the tail past the last whole wave is split in
        two when those units fit in one wave (else nothing is split);
      * fewer tiles than SM pairs (e.g. the 512-row A block of an 8-GPU
        strong-scaled 4096^3 sgemm: 32 tiles on 74 pairs): every tile is split
        in S = min(4, pairs // tiles) K ranges (persistent kernel only).
    Each K range keeps >= 2 K blocks of 32.  RISE_GEMM_KSPLIT=0 disables it."""
    tiles = pair_tiles(M, N, bn)
    slots = max(1, sm // 2)
    kb = -(-K // 32)
    if os.environ.get("RISE_GEMM_KSPLIT", "1") != "1" or tiles == 0 or kb < 2:
        return tiles, 1
    if tiles < slots:
        s = min(4, slots // tiles, kb // 2) if persistent else 1
        while s > 1 and tiles * (s - 1) > SPLIT_SLOTS_MAX:  # the parked parts' workspace
            s -= 1
        return (0, s) if s >= 2 else (tiles, 1)
    tail = tiles % slots
    if tail == 0 or 2 * tail > slots or tail > SPLIT_SLOTS_MAX:
        return tiles, 1
    return tiles - tail, 2


def full_tiles(M, N, K, bn, sm):
    """How many 256 x bn pair tiles run whole (schedule())."""
    return schedule(M, N, K, bn, sm)[0]


def work_units(M, N, K, bn, sm):
    nfull, s = schedule(M, N, K, bn, sm)
    return nfull + s * (pair_tiles(M, N, bn) - nfull)


def launch(st, nats, sm):
    from .emit_cuda import eval_py

    M = eval_py(st["M"], nats)
    N = eval_py(st["N"], nats)
    if st.get("pair"):
        K = eval_py(st["K"], nats)
        nfull, s = schedule(M, N, K, st["bn"], sm, st.get("persistent", False))
        if not st.get("persistent") and s != 2:
            nfull = pair_tiles(M, N, st["bn"])  # the non-persistent kernel splits tail tiles in two only
        units = nfull + max(s, 2) * (pair_tiles(M, N, st["bn"]) - nfull)
        if st.get("persistent"):  # one pair per SM pair, looping over the units
            return (2 * max(1, min(units, sm // 2)), 1, 1), (320, 1, 1), st["smem"], (2, 1, 1)
        return (2 * units, 1, 1), (192, 1, 1), st["smem"], (2, 1, 1)
    return (N // st["bn"], M // 128, 1), (192, 1, 1), st["smem"], (1, 1, 1)
