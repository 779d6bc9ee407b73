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
    loops, body = parallel_rows(stage)
    if loops is None or len(loops) != 2 or stage.kind != "grid":
        return None
    (iv, M), (jv, N) = loops
    shape = fold_shape(body)
    if shape is None:
        return None
    acc, init, loop, post = shape
    if not (isinstance(init.value, lir.Lit) and init.value.text in ("0.0f", "0f", "0.0")):
        return None
    p, K = loop.var, loop.bound
    step = loop.body.value
    if not (isinstance(step, lir.Bin) and step.op == "+" and step.a == acc and isinstance(step.b, lir.Bin)
            and step.b.op == "*" and isinstance(step.b.a, lir.Load) and isinstance(step.b.b, lir.Load)
            and step.ctype == "float"):
        return None
    x, y = step.b.a, step.b.b
    V = nat.Var

    def is_row(ld, var):
        return nat.equal(ld.index, nat.normalize(V(var) * K + V(p)), prog.assumptions)

    def is_col(ld, var):  # B[k][j] of a row-major K x N matrix (e.g. read through transpose(B))
        return nat.equal(ld.index, nat.normalize(V(p) * N + V(var)), prog.assumptions)

    b_mn = False  # B is MN-major in shared memory (UMMA b_major = 1)
    if is_row(x, iv) and is_row(y, jv):
        a_ld, b_ld = x, y
    elif is_row(y, iv) and is_row(x, jv):
        a_ld, b_ld = y, x
    elif PAIR and is_row(x, iv) and is_col(y, jv):
        a_ld, b_ld, b_mn = x, y, True
    elif PAIR and is_row(y, iv) and is_col(x, jv):
        a_ld, b_ld, b_mn = y, x, True
    else:
        return None
    for ld in (a_ld, b_ld):
        if prog.buffers[ld.buf].role != "input":
            return None
    if len(post) != 1:
        return None
    st = post[0]
    if not (isinstance(st, lir.Assign) and isinstance(st.target, lir.Store) and st.value == acc
            and nat.equal(st.target.index, nat.normalize(V(iv) * N + V(jv)), prog.assumptions)):
        return None
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
            f"({st.target.buf}, {r(N)}, &rs_mapA, &rs_mapB, {args});",
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
                {"kind": "tma2d", "buf": a_ld.buf, "offset": "0", "dims": [py_expr(K), py_expr(M)],
                 "pitch": py_expr(K), "box": [32, 128], "swizzle": 3},
                ({"kind": "tma2d", "buf": b_ld.buf, "offset": "0", "dims": [py_expr(N), py_expr(K)],
                  "pitch": py_expr(N), "box": [32, 32], "swizzle": 4} if b_mn else
                 {"kind": "tma2d", "buf": b_ld.buf, "offset": "0", "dims": [py_expr(K), py_expr(N)],
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
                          {"name": f"rs_ws_{base_name}_kflags", "ctype": "int", "size": "2 * 74"}],
        }
        return "\n".join(lines) + "\n", plan
    lines += [
        f"  rise_gemm::gemm_3xtf32<{r(K)}, {bn}, {stages}, {'true' if write_hi else 'false'}>"
        f"({st.target.buf}, {r(N)}, &rs_mapA, &rs_mapB);",
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
            {"kind": "tma2d", "buf": a_ld.buf, "offset": "0", "dims": [py_expr(K), py_expr(M)], "pitch": py_expr(K),
             "box": [32, 128], "swizzle": 3},
            {"kind": "tma2d", "buf": b_ld.buf, "offset": "0", "dims": [py_expr(K), py_expr(N)], "pitch": py_expr(K),
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
