"""`seqfold` template: a top-level sequential fold kept in the program's order.

Matches a serial stage of the form

    acc = INIT
    for j < K:  acc = STEP(acc, B1[c1 + j], B2[c2 + j], ...)   (unit-stride loads)
    POST(acc)

(the second stage of the chunked dot, or any `reduceSeq` emitted with
reassociate=False).  The dependent chain of K adds cannot be parallelised
without reordering, so the template makes the chain the only cost: one lane
streams 2048-element tiles of every stream into a 3-stage shared-memory ring
with 1-D bulk copies (TMA; the next tiles are in flight while the current
one is folded, and the lane never waits on a global load) and runs the
program's own step expression over float4 reads of shared memory, so the
chain advances at the FADD latency (full tiles: a register pipeline loads
the next 16 elements while the current 16 are folded).  Order: PRESERVED (bit-exact).
"""

from __future__ import annotations

import os

from . import lir
from ._ref import nat
from .emit_cuda import NatRenderer, ValueRenderer, kernel_head, py_expr

TILE = int(os.environ.get("RISE_SEQFOLD_TILE", "2048"))  # floats per stage (split among the streams: static smem < 48 KB)
STAGES = 3


def match(prog, stage, base_name, temps, exact, fold_shape, j_coefficient, thread_lines):
    if stage.kind != "serial":
        return None
    shape = fold_shape(stage.stmt)
    if shape is None:
        return None
    acc, init, loop, post = shape
    j = loop.var
    step = loop.body.value
    streams = {}
    for ld in dict.fromkeys(lir.expr_loads(step)):
        if any(v in prog.clamps for v in nat.free_vars(ld.index)):
            return None
        coef, base = j_coefficient(ld.index, j)
        if coef is None:
            return None
        if coef == 0:
            if not nat.free_vars(ld.index) <= set(prog.nat_params):
                return None
            continue
        if not nat.free_vars(base) <= set(prog.nat_params) or prog.buffers[ld.buf].ctype != "float":
            return None
        if prog.buffers[ld.buf].role == "pointer":
            return None
        streams[ld] = (ld.buf, base)
    if not streams:
        return None
    s_list = list(dict.fromkeys(streams.values()))
    r = NatRenderer(prog.clamps)
    name = f"{base_name}_seqfold"
    ns = len(s_list)

    def step_with(comp):
        def hook(ld):
            if ld in streams:
                return f"rs_v{s_list.index(streams[ld])}.{comp}" if comp else \
                    f"rs_ring[rs_q][{s_list.index(streams[ld])}][rs_jj]"
            return None

        return ValueRenderer(prog, exact, load_hook=hook)(step)

    pre = [f"({py_expr(base)}) % 4 == 0" for _b, base in s_list]
    lines = kernel_head(prog, name, temps, launch_bounds=32)
    lines += [
        f"  constexpr int RS_K = {r(loop.bound)};",
        f"  constexpr int RS_TILE = {max(256, TILE // ns)}, RS_S = {STAGES}, RS_NS = {ns};",
        "  constexpr int RS_NT = (RS_K + RS_TILE - 1) / RS_TILE;",
        "  // +16: the register pipeline below reads one group past a full tile (never used)",
        "  __shared__ __align__(128) float rs_ring[RS_S][RS_NS][RS_TILE + 16];",
        "  __shared__ __align__(8) unsigned long long rs_bar[RS_S];",
    ]
    for k, (buf, base) in enumerate(s_list):
        lines.append(f"  const float* rs_g{k} = {buf} + ({r(base)});")
    lines += [
        "  if (threadIdx.x != 0) return;  // the fold is one dependent chain: one lane runs it",
        "  for (int rs_q = 0; rs_q < RS_S; ++rs_q) rs_mbar_init(&rs_bar[rs_q], 1);",
        "  rs_fence_barrier_init();",
        "  // tile t -> stage t % S by 1-D bulk copies (TMA); the tail of K % 4 elements is read directly",
        "  constexpr int RS_K4 = RS_K / 4 * 4;",
        "  auto rs_issue = [&](int rs_t) {",
        "    const int rs_j0 = rs_t * RS_TILE;",
        "    const int rs_n4 = RS_K4 - rs_j0 < RS_TILE ? RS_K4 - rs_j0 : RS_TILE;",
        "    if (rs_n4 <= 0) return;",
        "    const int rs_q = rs_t % RS_S;",
        "    rs_mbar_arrive_expect_tx(&rs_bar[rs_q], (unsigned)(rs_n4 * 4 * RS_NS));",
    ]
    for k in range(ns):
        lines.append(f"    rs_bulk_g2s(rs_ring[rs_q][{k}], rs_g{k} + rs_j0, (unsigned)(rs_n4 * 4), &rs_bar[rs_q]);")
    lines += [
        "  };",
        "  for (int rs_t = 0; rs_t < RS_S - 1 && rs_t < RS_NT; ++rs_t) rs_issue(rs_t);",
        f"  {acc.ctype} {acc.name} = {ValueRenderer(prog, exact)(init.value)};",
        "  for (int rs_t = 0; rs_t < RS_NT; ++rs_t) {",
        "    if (rs_t + RS_S - 1 < RS_NT) {  // its stage was folded (generic-proxy reads) at t - 1",
        "      rs_fence_proxy_async();",
        "      rs_issue(rs_t + RS_S - 1);",
        "    }",
        "    const int rs_q = rs_t % RS_S;",
        "    const int rs_j0 = rs_t * RS_TILE;",
        "    const int rs_n4 = RS_K4 - rs_j0 < RS_TILE ? (RS_K4 - rs_j0 > 0 ? RS_K4 - rs_j0 : 0) : RS_TILE;",
        "    if (rs_n4 > 0) rs_mbar_wait(&rs_bar[rs_q], (unsigned)((rs_t / RS_S) & 1));",
        "    if (rs_n4 == RS_TILE) {",
        "      // full tile: the next 16 elements of every stream are loaded while the",
        "      // current 16 are folded, so the chain never waits on shared memory",
    ]
    ld = "*reinterpret_cast<const float4*>(&rs_ring[rs_q][{k}][{i}])"
    for k in range(ns):
        for u in range(4):
            lines.append(f"      float4 rs_c{k}_{u} = {ld.format(k=k, i=4 * u)};")
    lines += [
        "#pragma unroll 2",
        "      for (int rs_jj = 0; rs_jj < RS_TILE; rs_jj += 16) {",
    ]
    for k in range(ns):
        for u in range(4):
            lines.append(f"        const float4 rs_n{k}_{u} = {ld.format(k=k, i=f'rs_jj + {16 + 4 * u}')};")
    for u in range(4):
        lines.append("        {")
        for k in range(ns):
            lines.append(f"          const float4 rs_v{k} = rs_c{k}_{u};")
        for comp in ("x", "y", "z", "w"):
            lines.append(f"          {acc.name} = {step_with(comp)};")
        lines.append("        }")
    for k in range(ns):
        for u in range(4):
            lines.append(f"        rs_c{k}_{u} = rs_n{k}_{u};")
    lines += [
        "      }",
        "    } else {",
        "#pragma unroll 4",
        "    for (int rs_jj = 0; rs_jj < rs_n4; rs_jj += 4) {",
    ]
    for k in range(ns):
        lines.append(f"      const float4 rs_v{k} = *reinterpret_cast<const float4*>(&rs_ring[rs_q][{k}][rs_jj]);")
    for comp in ("x", "y", "z", "w"):
        lines.append(f"      {acc.name} = {step_with(comp)};")
    lines += [
        "    }",
        "    }",
        "  }",
        "  for (int rs_j = RS_K4; rs_j < RS_K; ++rs_j) {  // K % 4 tail, straight from global memory",
    ]
    for k in range(ns):
        lines.append(f"    const float4 rs_v{k} = make_float4(rs_g{k}[rs_j], 0.0f, 0.0f, 0.0f);")
    lines += [
        f"    {acc.name} = {step_with('x')};",
        "  }",
    ]
    for s_ in post:
        lines += ["  " + x for x in thread_lines(prog, s_, exact)]
    lines += ["}"]
    plan = {"name": name, "kind": "seqfold", "fmad": False, "order": "preserved", "pre": pre}
    return "\n".join(lines) + "\n", plan


def launch(st, nats, sm):
    return (1, 1, 1), (32, 1, 1), 0, (1, 1, 1)
