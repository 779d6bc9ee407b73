"""`transpose2d` template: a 2-D parallel map whose body reads a 2-D input
TRANSPOSED — the layout programs of SURVEY.md §8 a14 (`transpose`, and any
elementwise body over a transposed view).

Matches a stage whose parallel loops collapse to two variables (r < R,
c < C; the output is written along c) with no sequential loops in the
body, and in which some float input is loaded at  base + r + c * P  (unit
stride along r, a pitch P along c).  The generic kernel reads those loads
with a stride of P floats between neighbouring threads: one 32-byte sector
per 4-byte value, ≈ 1.9 TB/s at 8192² (`tools/probe_transpose.py`).

Data movement: a block owns a 128 x 128 output tile.  The TMA engine loads
the tile's input footprint — 128 rows of the input (c) x 128 columns (r),
as four [128 x 32-float] boxes with the 128-byte swizzle, 512 contiguous
bytes per input row — into shared memory; each thread then reads four
consecutive r of one c as one LDS.128 (the swizzle makes 8 consecutive
lanes = 8 consecutive c hit 8 different 16-byte chunks: conflict-free) and
computes the program's own body for those four outputs, whose stores are
coalesced along c (a warp writes 128 contiguous bytes of each output row).

Order: PRESERVED — each output is the program's body on the same values.
Bit-identical to the reference's semantics.
"""

from __future__ import annotations

from . import lir
from ._ref import nat
from .emit_cuda import GenericKernel, NatRenderer, Stage, ValueRenderer, kernel_head, py_expr

T = 128  # output tile: T rows (r) x T columns (c)
BOX = 32  # floats per swizzled box row (128 bytes)
BLOCK = 256


def _affine2(index, rv, cv, params):
    """index = base + a * rv + b * cv with base, a, b free of rv / cv (sizes
    only): (base, a, b), else None."""
    def at(r, c):
        return nat.normalize(nat.substitute(index, {rv: nat.Const(r), cv: nat.Const(c)}))

    base = at(0, 0)
    a, b = nat.normalize(at(1, 0) - base), nat.normalize(at(0, 1) - base)
    if not nat.equal(nat.normalize(at(2, 0) - base), nat.normalize(a * nat.Const(2))):
        return None
    if not nat.equal(nat.normalize(at(0, 2) - base), nat.normalize(b * nat.Const(2))):
        return None
    if not nat.equal(nat.normalize(at(1, 1) - base), nat.normalize(a + b)):
        return None
    for e in (base, a, b):
        if not nat.free_vars(e) <= set(params):
            return None
    return base, a, b


def match(prog, stage, base_name, temps, exact, parallel_rows):
    if stage.kind != "grid":
        return None
    loops, body = parallel_rows(stage)
    if loops is None or len(loops) != 2:
        return None
    (rv, R), (cv, C) = loops
    for t in lir.walk(body):
        if isinstance(t, (lir.For, lir.ParFor, lir.DoubleBuffer, lir.Alloc)):
            return None
    params = list(prog.nat_params)
    streams = {}  # load -> (buf, base, pitch)
    for _t, value in lir.stmt_exprs(body):
        for ld in lir.expr_loads(value):
            if any(v in prog.clamps for v in nat.free_vars(ld.index)):
                return None
            if rv not in nat.free_vars(ld.index):
                continue
            aff = _affine2(ld.index, rv, cv, params)
            if aff is None:
                return None
            base, a, b = aff
            buf = prog.buffers[ld.buf]
            if (nat.equal(a, nat.Const(1)) and not isinstance(b, nat.Const) and buf.ctype == "float"
                    and buf.role == "input"):
                streams[ld] = (ld.buf, base, b)
    s_list = list(dict.fromkeys(streams.values()))
    if not s_list or len(s_list) > 2:
        return None
    r = NatRenderer(prog.clamps)
    name = f"{base_name}_transpose"
    ns = len(s_list)
    box_floats = T * BOX
    pre = [f"({py_expr(R)}) > 0", f"({py_expr(C)}) > 0"]
    tmaps = []
    for buf, base, pitch in s_list:
        # (16-byte aligned base and pitch; rows of the read region must not overlap: R <= P)
        pre += [f"({py_expr(base)}) % 4 == 0", f"({py_expr(pitch)}) % 4 == 0", f"({py_expr(pitch)}) >= ({py_expr(R)})"]
        tmaps.append({"kind": "tma2d", "buf": buf, "offset": py_expr(base), "dims": [py_expr(R), py_expr(C)],
                      "pitch": py_expr(pitch), "box": [BOX, T], "swizzle": 3})
    pre = list(dict.fromkeys(pre))

    def body_for(q):
        def hook(ld):
            if ld in streams:
                return f"rs_v{s_list.index(streams[ld])}.{'xyzw'[q]}"
            return None

        g = GenericKernel(prog, Stage("serial", body), "_", [], exact)
        g.r = ValueRenderer(prog, exact, load_hook=hook)
        return g.thread(body, 4)

    extra = [f"const __grid_constant__ rs_tmap rs_map{k}" for k in range(ns)]
    lines = kernel_head(prog, name, temps, launch_bounds=BLOCK, extra_params=extra)
    lines += [
        f"  constexpr int RS_R = {r(R)}, RS_C = {r(C)}, RS_T = {T}, RS_BOXF = {box_floats};",
        "  extern __shared__ __align__(1024) unsigned char rs_smem_raw[];",
        "  float* rs_smem = reinterpret_cast<float*>(rs_smem_raw + ((1024u - (rs_smem_addr(rs_smem_raw) & 1023u)) & 1023u));",
        f"  unsigned long long* rs_bar = reinterpret_cast<unsigned long long*>(rs_smem + {ns * 4} * RS_BOXF);",
        "  const int rs_r0 = blockIdx.y * RS_T, rs_c0 = blockIdx.x * RS_T;",
        "  if (threadIdx.x == 0) {",
        "    rs_mbar_init(rs_bar, 1);",
        "    rs_fence_barrier_init();",
        f"    rs_mbar_arrive_expect_tx(rs_bar, (unsigned)({ns * 4} * RS_BOXF * 4));  // (out-of-range cells arrive as 0)",
    ]
    for k in range(ns):
        lines.append(f"    for (int rs_b = 0; rs_b < 4; ++rs_b) "
                     f"rs_tma_load_2d(rs_smem + ({k * 4} + rs_b) * RS_BOXF, &rs_map{k}, rs_r0 + {BOX} * rs_b, rs_c0, rs_bar);")
    lines += [
        "  }",
        "  __syncthreads();",
        "  rs_mbar_wait(rs_bar, 0);",
        "  // warp w: tile columns (w & 3) * 32 + lane, tile rows (w >> 2) * 64 .. + 63, four at a time",
        "  const int rs_cl = ((threadIdx.x >> 5) & 3) * 32 + (threadIdx.x & 31);",
        "  const int rs_rh = (threadIdx.x >> 7) * 64;",
        f"  const int {cv} = rs_c0 + rs_cl;",
        "#pragma unroll 2",
        "  for (int rs_k = 0; rs_k < 16; ++rs_k) {",
        "    const int rs_rl = rs_rh + 4 * rs_k;",
        f"    const int rs_off = ((rs_rl >> 5) * RS_T + rs_cl) * {BOX} + ((((rs_rl & 31) >> 2) ^ (rs_cl & 7)) << 2);",
    ]
    for k in range(ns):
        lines.append(f"    const float4 rs_v{k} = *reinterpret_cast<const float4*>(rs_smem + {k * 4} * RS_BOXF + rs_off);")
    for q in range(4):
        lines += [
            "    {",
            f"      const int {rv} = rs_r0 + rs_rl + {q};",
            f"      if ({rv} < RS_R && {cv} < RS_C) {{",
        ]
        lines += ["    " + x for x in body_for(q)]
        lines += ["      }", "    }"]
    lines += ["  }", "}"]
    smem = ns * 4 * box_floats * 4 + 1024 + 16
    plan = {
        "name": name,
        "kind": "transpose2d",
        "rows": py_expr(R),
        "cols": py_expr(C),
        "block": BLOCK,
        "smem": smem,
        "fmad": False,
        "order": "preserved",
        "pre": pre,
        "extra_args": tmaps,
    }
    return "\n".join(lines) + "\n", plan


def launch(st, nats, sm):
    from .emit_cuda import eval_py

    rows, cols = eval_py(st["rows"], nats), eval_py(st["cols"], nats)
    return (max(1, -(-cols // T)), max(1, -(-rows // T)), 1), (st["block"], 1, 1), st["smem"], (1, 1, 1)
