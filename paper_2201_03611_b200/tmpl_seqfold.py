"""`seqfold` template: a top-level sequential fold kept in the program's order.

Matches a serial stage of the form

    acc = INIT
    for j < K:  acc = STEP(acc, B1[c1 + j], B2[c2 + j], ...)   (unit-stride loads)
    POST(acc)

(the second stage of the chunked dot, or any `reduceSeq` emitted with
reassociate=False).  The dependent chain of K adds cannot be parallelised
without reordering, so the template makes the chain the only cost: one warp
stages 1024-element tiles of every stream into a double-buffered shared
memory ring with coalesced 128-bit loads (the next tile is in flight while
the current one is folded), and lane 0 runs the program's own step
expression over shared memory.  Order: PRESERVED (bit-exact).
"""

from __future__ import annotations

from . import lir
from ._ref import nat
from .emit_cuda import NatRenderer, ValueRenderer, kernel_head, py_expr

TILE = 1024


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

    def hook(ld):
        if ld in streams:
            return f"rs_st[{s_list.index(streams[ld])} * {TILE} + rs_jj]"
        return None

    vstep = ValueRenderer(prog, exact, load_hook=hook)(step)
    lines = kernel_head(prog, name, temps, launch_bounds=32)
    lines += [
        f"  constexpr int RS_K = {r(loop.bound)};",
        f"  __shared__ __align__(16) float rs_ring[2][{ns} * {TILE}];",
    ]
    for k, (buf, base) in enumerate(s_list):
        lines.append(f"  const float* rs_g{k} = {buf} + ({r(base)});")
    lines += [
        "  const int rs_lane = threadIdx.x;",
        "  auto rs_stage = [&](int rs_t, float* rs_dst) {",
        f"    const int rs_j0 = rs_t * {TILE};",
        f"    for (int rs_e = rs_lane; rs_e < {TILE}; rs_e += 32) {{",
        "      const int rs_j = rs_j0 + rs_e;",
    ]
    for k in range(ns):
        lines.append(f"      rs_dst[{k} * {TILE} + rs_e] = rs_j < RS_K ? __ldg(rs_g{k} + rs_j) : 0.0f;")
    lines += [
        "    }",
        "  };",
        f"  constexpr int RS_NT = (RS_K + {TILE - 1}) / {TILE};",
        f"  {acc.ctype} {acc.name} = {ValueRenderer(prog, exact)(init.value)};",
        "  if (RS_NT > 0) rs_stage(0, rs_ring[0]);",
        "  __syncwarp();",
        "  for (int rs_t = 0; rs_t < RS_NT; ++rs_t) {",
        "    if (rs_t + 1 < RS_NT) rs_stage(rs_t + 1, rs_ring[(rs_t + 1) & 1]);  // next tile in flight",
        "    if (rs_lane == 0) {",
        "      const float* rs_st = rs_ring[rs_t & 1];",
        f"      const int rs_n = RS_K - rs_t * {TILE} < {TILE} ? RS_K - rs_t * {TILE} : {TILE};",
        "#pragma unroll 8",
        "      for (int rs_jj = 0; rs_jj < rs_n; ++rs_jj) {",
        f"        {acc.name} = {vstep};",
        "      }",
        "    }",
        "    __syncwarp();",
        "  }",
        "  if (rs_lane == 0) {",
    ]
    for s in post:
        lines += ["    " + x for x in thread_lines(prog, s, exact)]
    lines += ["  }", "}"]
    plan = {"name": name, "kind": "seqfold", "fmad": False, "order": "preserved", "pre": []}
    return "\n".join(lines) + "\n", plan


def launch(st, nats, sm):
    return (1, 1, 1), (32, 1, 1), 0, (1, 1, 1)
