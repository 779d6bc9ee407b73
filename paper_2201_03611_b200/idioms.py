"""Idiom matching: LIR stages -> hand-written sm_100a kernel templates.

A template is chosen only when the stage's loop nest has exactly the shape
the template implements; otherwise the generic kernel (emit_cuda.py) runs.
Each template keeps or states the program's evaluation order:

* `rowfold` (tmpl_rowfold.py) — a parallel map over rows whose body is a
  sequential fold over j with unit-stride loads (gemv `mv.rise`, the paper's
  `mv_opt` schedule, chunked reductions).  Order PRESERVED (bit-exact); TMA
  streams the rows through swizzled shared memory.
* `reduce` — a top-level sequential fold `acc = acc + term(i)` over the
  whole input (the `dot` program after `toReduceSeq`).  One chain of 2^24
  dependent adds cannot run in parallel in its own order, so this template
  REASSOCIATES `+` into a fixed, documented tree (DESIGN.md "Reduction
  order"): per-thread left folds over a fixed strided float4 partition, a
  warp butterfly, a block butterfly, and a last-block fold of the block
  partials.  The order depends only on the problem size, never on the GPU
  or on scheduling; parity is the fp64 error bound of SURVEY.md §8 d.
* `stencil2d`, `allpairs`, `gemm_tc` — see their modules.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from . import lir, tmpl_allpairs, tmpl_gemm, tmpl_gridseq, tmpl_iterate, tmpl_rowfold, tmpl_seqfold, tmpl_stencil, tmpl_stencil1d, tmpl_transpose
from ._ref import nat
from .emit_cuda import NatRenderer, ValueRenderer, collapse_global_chain, kernel_head, py_expr


@dataclass
class IdiomKernel:
    name: str
    text: str
    plan: dict
    includes: list = field(default_factory=list)


ORDER_PRESERVING = ("_match_rowfold", "_match_stencil", "_match_seqfold", "_match_iterate", "_match_transpose",
                    "_match_stencil1d", "_match_gridseq")


def _match_iterate(prog, stage, base_name, temps, exact):
    out = tmpl_iterate.match(prog, stage, base_name, temps, exact)
    if out is None:
        return None
    text, plan = out
    return IdiomKernel(plan["name"], text, plan)


def _match_gridseq(prog, stage, base_name, temps, exact):
    out = tmpl_gridseq.match(prog, stage, base_name, temps, exact)
    if out is None:
        return None
    text, plan = out
    return IdiomKernel(plan["name"], text, plan)


def _match_seqfold(prog, stage, base_name, temps, exact):
    out = tmpl_seqfold.match(prog, stage, base_name, temps, exact, fold_shape, j_coefficient, thread_lines)
    if out is None:
        return None
    text, plan = out
    return IdiomKernel(plan["name"], text, plan)


def match(prog, stage, base_name, temps, exact, reassociate=True):
    for matcher in (_match_gemm, _match_gemm_tiled, _match_rowfold, _match_reduce, _match_stencil, _match_allpairs,
                    _match_seqfold, _match_iterate, _match_transpose, _match_stencil1d, _match_gridseq):
        if not reassociate and matcher.__name__ not in ORDER_PRESERVING:
            continue
        out = matcher(prog, stage, base_name, temps, exact)
        if out is not None:
            return out
    return None


def _match_gemm(prog, stage, base_name, temps, exact):
    out = tmpl_gemm.match(prog, stage, base_name, temps, exact, parallel_rows, fold_shape)
    if out is None:
        return None
    text, plan = out
    return IdiomKernel(plan["name"], text, plan, includes=["rise/gemm_tc.cuh"])


def _match_gemm_tiled(prog, stage, base_name, temps, exact):
    """The tiled sgemm program (programs.SGEMM_TILED): workgroups over row
    blocks of A staged in Local memory, work-items over columns, K in tiles —
    recognised as the same contraction and run on the tensor cores."""
    out = tmpl_gemm.match_tiled(prog, stage, base_name, temps, exact, fold_shape)
    if out is None:
        return None
    text, plan = out
    return IdiomKernel(plan["name"], text, plan, includes=["rise/gemm_tc.cuh"])


def _match_allpairs(prog, stage, base_name, temps, exact):
    out = tmpl_allpairs.match(prog, stage, base_name, temps, exact, parallel_rows)
    if out is None:
        return None
    text, plan = out
    return IdiomKernel(plan["name"], text, plan)


def _match_stencil1d(prog, stage, base_name, temps, exact):
    out = tmpl_stencil1d.match(prog, stage, base_name, temps, exact, parallel_rows)
    if out is None:
        return None
    text, plan = out
    return IdiomKernel(plan["name"], text, plan)


def _match_transpose(prog, stage, base_name, temps, exact):
    out = tmpl_transpose.match(prog, stage, base_name, temps, exact, parallel_rows)
    if out is None:
        return None
    text, plan = out
    return IdiomKernel(plan["name"], text, plan)


def _match_stencil(prog, stage, base_name, temps, exact):
    out = tmpl_stencil.match(prog, stage, base_name, temps, exact, parallel_rows)
    if out is None:
        return None
    text, plan = out
    return IdiomKernel(plan["name"], text, plan)


# ---------------------------------------------------------------------------
# shared analysis helpers


def parallel_rows(stage):
    """Collapse the stage's parallel loops into rows: ([(var, bound)], body)."""
    s = stage.stmt
    if stage.kind == "grid":
        return collapse_global_chain(s)
    if stage.kind == "workgroup":
        loops = [(s.var, s.bound)]
        body = s.body
        if isinstance(body, lir.ParFor) and body.kind == "local":
            loops.append((body.var, body.bound))
            return loops, body.body
    return None, None


def fold_shape(body):
    """Alloc(acc scalar) { acc = INIT; for j < K: acc = STEP; POST... }"""
    if not (isinstance(body, lir.Alloc) and body.dims == () and body.space == "Private"):
        return None
    acc = lir.ScalarRef(body.name, body.ctype)
    stmts = body.body.stmts if isinstance(body.body, lir.Seq) else [body.body]
    if len(stmts) < 2:
        return None
    init, loop, post = stmts[0], stmts[1], stmts[2:]
    if not (isinstance(init, lir.Assign) and init.target == acc):
        return None
    if acc in set(lir.expr_scalars(init.value)):
        return None
    if not (isinstance(loop, lir.For) and isinstance(loop.body, lir.Assign) and loop.body.target == acc):
        return None
    for s in post:
        for t in lir.walk(s):
            if isinstance(t, (lir.For, lir.ParFor, lir.DoubleBuffer, lir.Alloc)):
                return None
    return acc, init, loop, post


def j_coefficient(index, j):
    """0 if `index` does not use j, 1 if index == base + j, else None."""
    if j not in nat.free_vars(index):
        return 0, index
    base = nat.normalize(nat.substitute(index, {j: nat.Const(0)}))
    if nat.equal(nat.normalize(base + nat.Var(j)), nat.normalize(index)) and j not in nat.free_vars(base):
        return 1, base
    return None, None


def uses_clamp(n, prog):
    return any(v in prog.clamps for v in nat.free_vars(n))


def thread_lines(prog, stmt, exact):
    from .emit_cuda import GenericKernel, Stage

    return GenericKernel(prog, Stage("serial", stmt), "_", [], exact).thread(stmt, 0)


# ---------------------------------------------------------------------------
# rowfold


def _match_rowfold(prog, stage, base_name, temps, exact):
    loops, body = parallel_rows(stage)
    if loops is None:
        return None
    shape = fold_shape(body)
    if shape is None:
        return None
    acc, init, loop, post = shape
    j = loop.var
    row_vars = [v for v, _ in loops]
    step = loop.body.value
    row_streams, shared_streams = {}, {}
    allowed = set(row_vars) | set(prog.nat_params)
    for ld in dict.fromkeys(lir.expr_loads(step)):
        if uses_clamp(ld.index, prog):
            return None
        coef, base = j_coefficient(ld.index, j)
        if coef is None:
            return None
        if coef == 0:
            if not nat.free_vars(ld.index) <= allowed:
                return None
            continue  # j-invariant: read directly from global memory
        buf = prog.buffers[ld.buf]
        if buf.role == "pointer" or (buf.role == "alloc" and buf.space != "Global"):
            return None
        if not nat.free_vars(base) <= allowed:
            return None
        if any(v in nat.free_vars(base) for v in row_vars):
            row_streams[ld] = (ld.buf, base)
        else:
            shared_streams[ld] = (ld.buf, base)
    if not row_streams:
        return None
    if any(prog.buffers[b].ctype != "float" for b, _ in list(row_streams.values()) + list(shared_streams.values())):
        return None  # the staging moves fp32 words (float4 views)
    name = f"{base_name}_rowfold"
    out = tmpl_rowfold.emit(prog, loops, shape, row_streams, shared_streams, name, temps, exact, j)
    if out is None:
        return None
    text, plan = out
    return IdiomKernel(name, text, plan)


def _launch_rowfold(st, nats, sm):
    from .emit_cuda import eval_py

    rows = eval_py(st["rows"], nats)
    rb = eval_py(str(st["row_block"]), nats)
    grid = max(1, -(-rows // rb))
    return (grid, 1, 1), (rb, 1, 1), eval_py(str(st["smem"]), nats), (1, 1, 1)


# ---------------------------------------------------------------------------
# reduce (reassociated, deterministic)

import os  # noqa: E402

# Fixed launch shape: the reduction order depends only on these constants and
# the problem size, never on the GPU.  (Overridable for tuning sweeps only.)
REDUCE_GRID = int(os.environ.get("RISE_REDUCE_GRID", "1184"))
REDUCE_BLOCK = int(os.environ.get("RISE_REDUCE_BLOCK", "256"))
REDUCE_BATCH = int(os.environ.get("RISE_REDUCE_BATCH", "8"))  # float4 chunks per input in flight per thread
# occupancy hint for __launch_bounds__ (never changes the order).  1: forcing
# the whole grid resident (8 blocks/SM) caps registers at 32 and spills the
# load batch — measured 2.0 TB/s instead of 4.6 at 2^24
REDUCE_MINB = int(os.environ.get("RISE_REDUCE_MINB", "1"))
# TMA variant (default): a fixed grid of REDUCE_TMA_GRID blocks (2 per SM on a
# 148-SM B200: one wave), each streaming its chunks (REDUCE_TMA_CHUNK bytes
# per input) through a REDUCE_TMA_STAGES-deep shared-memory ring filled by
# cp.async.bulk from one producer lane; the REDUCE_BLOCK folding threads only
# read shared memory.  Order: see DESIGN.md §4.
REDUCE_TMA = os.environ.get("RISE_REDUCE_TMA", "1") == "1"
# 256 blocks (measured at 2^24 on two boxes, profiles/dot_grid_r02c.txt:
# 256 0.944 / 0.966 against 296 0.930 / 0.950; 128-248 and 264-512 lower):
# 2^24 elements are 8192 chunks, exactly 32 per block
REDUCE_TMA_GRID = int(os.environ.get("RISE_REDUCE_TMA_GRID", "256"))
# measured (2^24, round-robin inputs, three passes on one box): 16 KiB x 3 stages
# 0.78, 8 KiB x 4 stages 0.82 (less shared memory, more chunks in flight)
REDUCE_TMA_CHUNK = int(os.environ.get("RISE_REDUCE_TMA_CHUNK", "8192"))
REDUCE_TMA_STAGES = int(os.environ.get("RISE_REDUCE_TMA_STAGES", "4"))
REDUCE_TMA_CONTIG = os.environ.get("RISE_REDUCE_TMA_CONTIG", "0") == "1"
# the producer lane fills the ring before the block-wide barrier (measured +0.5-1 %)
REDUCE_EARLY = os.environ.get("RISE_REDUCE_EARLY", "1") == "1"  # 2-D tensor-map boxes instead of bulk copies


def _reduce_tma_stages(nstreams: int) -> int:
    """Ring depth of the TMA variant for `nstreams` input streams (~200 KiB of
    shared memory); < 2 means the register-batched LDG variant is emitted."""
    return min(REDUCE_TMA_STAGES, (200 * 1024) // (nstreams * REDUCE_TMA_CHUNK))


def reduce_fold_length(n: int, streams: int = 2) -> int:
    """Terms one thread folds sequentially in phase 1 of the `reduce`
    template for n terms read from `streams` input streams (its error
    bound's sequential part)."""
    n4 = n // 4
    tail = n - 4 * n4  # folded after the float4 part by the last block
    if REDUCE_TMA and _reduce_tma_stages(streams) >= 2:
        ch4 = REDUCE_TMA_CHUNK // 16
        chunks = -(-n4 // ch4)
        return 4 * -(-chunks // REDUCE_TMA_GRID) * -(-ch4 // REDUCE_BLOCK) + tail
    return 4 * -(-n4 // (REDUCE_GRID * REDUCE_BLOCK)) + tail


def _match_reduce(prog, stage, base_name, temps, exact):
    if stage.kind != "serial":
        return None
    shape = fold_shape(stage.stmt)
    if shape is None:
        return None
    acc, init, loop, post = shape
    step = loop.body.value
    if not (isinstance(step, lir.Bin) and step.op == "+" and step.a == acc):
        return None
    term = step.b
    if acc in set(lir.expr_scalars(term)):
        return None
    i = loop.var
    streams = {}
    for ld in dict.fromkeys(lir.expr_loads(term)):
        if uses_clamp(ld.index, prog):
            return None
        coef, base = j_coefficient(ld.index, i)
        if coef is None:
            return None
        if coef == 1:
            if not nat.free_vars(base) <= set(prog.nat_params):
                return None
            streams[ld] = (ld.buf, base)
        elif not nat.free_vars(ld.index) <= set(prog.nat_params):
            return None
    if not streams:
        return None
    if any(prog.buffers[b].ctype != "float" for b, _ in streams.values()):
        return None  # float4 streaming loads
    for s in post:  # post may only read the accumulator and write memory
        for t in lir.walk(s):
            if isinstance(t, lir.Assign) and isinstance(t.target, lir.ScalarRef) and t.target != acc:
                return None
    pre = []  # any n: the n % 4 tail is folded by the last block (below)
    for _b, base in streams.values():
        pre.append(f"({py_expr(base)}) % 4 == 0")
    pre = list(dict.fromkeys(pre))
    s_list = list(dict.fromkeys(streams.values()))
    name = f"{base_name}_reduce"
    r = NatRenderer(prog.clamps)
    ct = acc.ctype
    zero = "0.0f" if ct == "float" else "0"
    vr_plain = ValueRenderer(prog, exact)

    def add(a, b):
        return f"__fadd_rn({a}, {b})" if (ct == "float" and exact) else f"({a} + {b})"

    def to_bits(v):
        return f"__float_as_uint({v})" if ct == "float" else f"(unsigned)({v})"

    def from_bits(v):
        return f"__uint_as_float({v})" if ct == "float" else f"(int)({v})"

    def term_with(u, comp):
        def hook(ld):
            if ld in streams:
                return f"rs_v{s_list.index(streams[ld])}[{u}].{comp}"
            return None

        return ValueRenderer(prog, exact, load_hook=hook)(term)

    def tail_hook(ld):
        if ld in streams:
            buf, base = streams[ld]
            return f"{buf}[({r(base)}) + rs_j]"
        return None

    tail_term = ValueRenderer(prog, exact, load_hook=tail_hook)(term)
    shfl = "__shfl_xor_sync(0xffffffffu, rs_s, rs_o)"
    U = REDUCE_BATCH
    s_list = list(dict.fromkeys(streams.values()))
    # many input streams: when not even a double-buffered TMA ring fits, the
    # register-batched LDG variant (any number of streams) is emitted instead
    tma = REDUCE_TMA and _reduce_tma_stages(len(s_list)) >= 2
    B = REDUCE_BLOCK  # threads that fold (the TMA variant adds one producer warp)
    G = REDUCE_TMA_GRID if tma else REDUCE_GRID
    nthreads = B + 32 if tma else B
    minb = REDUCE_MINB
    peers = int(getattr(prog, "peer_ranks", 0) or 0)
    if peers and not (tma and ct == "float"):
        return None
    # block partials as epoch-tagged 64-bit slots and a 64-bit launch counter
    # (no fence on the critical path: see phase 3 below)
    xparams = ["unsigned long long* __restrict__ rs_partials", "unsigned long long* __restrict__ rs_ticket"]
    if peers:
        # multi-GPU: the ranks' totals meet in peer memory (table: R slot arrays, then this rank)
        xparams += ["const unsigned long long* __restrict__ rs_xtab", "unsigned* __restrict__ rs_epoch"]
    lines = kernel_head(prog, name, temps, launch_bounds=f"{nthreads}, {minb}", extra_params=xparams)
    lines += [
        f"  constexpr int RS_N4 = ({r(loop.bound)}) / 4;",
        f"  constexpr int RS_G = {G}, RS_B = {B};",
    ]
    for k, (buf, base) in enumerate(s_list):
        lines.append(f"  const float4* __restrict__ rs_g{k} = reinterpret_cast<const float4*>({buf} + ({r(base)}));")
    lines.append(f"  {ct} rs_acc = {zero};")
    smem = 0
    if tma:
        NSTR = len(s_list)
        CH4 = REDUCE_TMA_CHUNK // 16
        # ring depth within ~200 KiB of shared memory (many input streams: fewer stages)
        S = _reduce_tma_stages(NSTR)
        smem = S * NSTR * CH4 * 16 + 2 * S * 8
        lines += [
            f"  constexpr int RS_CH4 = {CH4}, RS_S = {S}, RS_NSTR = {NSTR};",
            "  constexpr int RS_NCH = (RS_N4 + RS_CH4 - 1) / RS_CH4;",
            "  extern __shared__ __align__(128) unsigned char rs_smem_raw[];",
            "  float4* const rs_ring = reinterpret_cast<float4*>(rs_smem_raw);  // [stage][stream][RS_CH4]",
            "  unsigned long long* const rs_full = reinterpret_cast<unsigned long long*>(rs_ring + RS_S * RS_NSTR * RS_CH4);",
            "  unsigned long long* const rs_empty = rs_full + RS_S;",
        ]
        if REDUCE_TMA_CONTIG:
            lines += [
                "  // a contiguous run of chunks per block: [b*NCH/G, (b+1)*NCH/G) of RS_CH4 float4 per stream",
                "  const int rs_c0 = (int)(((long long)blockIdx.x * RS_NCH) / RS_G);",
                "  const int rs_nmine = (int)(((long long)(blockIdx.x + 1) * RS_NCH) / RS_G) - rs_c0;",
            ]
            chunk_of = "rs_c0 + rs_k"
        else:
            lines += [
                "  // chunks blockIdx.x, blockIdx.x + G, ... of RS_CH4 float4 per stream",
                "  const int rs_nmine = (int)blockIdx.x < RS_NCH ? (RS_NCH - 1 - (int)blockIdx.x) / RS_G + 1 : 0;",
            ]
            chunk_of = "(int)blockIdx.x + rs_k * RS_G"
        lines += [
            "  auto rs_issue = [&](int rs_k) {  // the producer lane: chunk rs_k of this block into its stage",
            "    const int rs_q = rs_k % RS_S;",
            f"    const int rs_c = {chunk_of};",
            "    const int rs_len = RS_N4 - rs_c * RS_CH4 < RS_CH4 ? RS_N4 - rs_c * RS_CH4 : RS_CH4;",
            "    rs_mbar_arrive_expect_tx(&rs_full[rs_q], (unsigned)(rs_len * 16 * RS_NSTR));",
        ]
        for k in range(NSTR):
            lines.append(f"    rs_bulk_g2s(rs_ring + (rs_q * RS_NSTR + {k}) * RS_CH4, rs_g{k} + (size_t)rs_c * RS_CH4, "
                         "(unsigned)(rs_len * 16), &rs_full[rs_q]);")
        lines += [
            "  };",
            "  if (threadIdx.x == RS_B) {",
            "    // the producer initialises the ring and fills it before the block-wide barrier",
            "    for (int rs_q = 0; rs_q < RS_S; ++rs_q) {",
            "      rs_mbar_init(&rs_full[rs_q], 1);",
            "      rs_mbar_init(&rs_empty[rs_q], RS_B / 32);",
            "    }",
            "    rs_fence_barrier_init();",
            f"    constexpr int RS_FIRST = {'RS_S' if REDUCE_EARLY else '0'};  // chunks issued before the barrier",
            "    for (int rs_k = 0; rs_k < RS_FIRST && rs_k < rs_nmine; ++rs_k) rs_issue(rs_k);",
            "  }",
            "  __syncthreads();",
            "  if (threadIdx.x >= RS_B) {",
            "    // producer warp: one lane streams the rest of the chunks through the ring (TMA)",
            "    if (threadIdx.x == RS_B) {",
            f"      for (int rs_k = {'RS_S' if REDUCE_EARLY else '0'}; rs_k < rs_nmine; ++rs_k) {{",
            "        if (rs_k >= RS_S) rs_mbar_wait(&rs_empty[rs_k % RS_S], ((rs_k / RS_S) & 1) ^ 1);",
            "        rs_issue(rs_k);",
            "      }",
            "    }",
            "  } else {",
            "    // phase 1: thread t folds, chunk after chunk, float4 t, t + B, t + 2B, ... of the chunk",
            "    for (int rs_k = 0; rs_k < rs_nmine; ++rs_k) {",
            "      const int rs_q = rs_k % RS_S;",
            f"      const int rs_c = {chunk_of};",
            "      const int rs_len = RS_N4 - rs_c * RS_CH4 < RS_CH4 ? RS_N4 - rs_c * RS_CH4 : RS_CH4;",
            "      rs_mbar_wait(&rs_full[rs_q], (rs_k / RS_S) & 1);",
            "#pragma unroll",
            "      for (int rs_i = 0; rs_i < (RS_CH4 + RS_B - 1) / RS_B; ++rs_i) {",
            "        const int rs_e = threadIdx.x + rs_i * RS_B;",
            "        if (rs_e < rs_len) {",
        ]
        for k in range(NSTR):
            lines.append(f"          const float4 rs_v{k}[1] = {{rs_ring[(rs_q * RS_NSTR + {k}) * RS_CH4 + rs_e]}};")
        for comp in ("x", "y", "z", "w"):
            lines.append(f"          rs_acc = {add('rs_acc', term_with('0', comp))};")
        lines += [
            "        }",
            "      }",
            "      __syncwarp();",
            "      if ((threadIdx.x & 31) == 0) rs_mbar_arrive(&rs_empty[rs_q]);",
            "    }",
            "  }",
        ]
    else:
        lines += [
            "  constexpr int RS_T = RS_G * RS_B;",
            "  constexpr int RS_ITERS = (RS_N4 + RS_T - 1) / RS_T;",
            "  const int rs_tid = blockIdx.x * blockDim.x + threadIdx.x;",
            "  // phase 1: thread-local left fold over float4 chunks tid, tid+T, tid+2T, ...",
            f"  for (int rs_it = 0; rs_it < RS_ITERS; rs_it += {U}) {{",
        ]
        for k in range(len(s_list)):
            lines.append(f"    float4 rs_v{k}[{U}];")
        lines += [
            "#pragma unroll",
            f"    for (int rs_u = 0; rs_u < {U}; ++rs_u) {{",
            "      const int rs_c = rs_tid + (rs_it + rs_u) * RS_T;",
            "      if (rs_it + rs_u < RS_ITERS && rs_c < RS_N4) {",
        ]
        for k in range(len(s_list)):
            lines.append(f"        rs_v{k}[rs_u] = rs_ldg_stream(rs_g{k} + rs_c);")
        lines += [
            "      }",
            "    }",
            "#pragma unroll",
            f"    for (int rs_u = 0; rs_u < {U}; ++rs_u) {{",
            "      const int rs_c = rs_tid + (rs_it + rs_u) * RS_T;",
            "      if (rs_it + rs_u < RS_ITERS && rs_c < RS_N4) {",
        ]
        for comp in ("x", "y", "z", "w"):
            lines.append(f"        rs_acc = {add('rs_acc', term_with('rs_u', comp))};")
        lines += [
            "      }",
            "    }",
            "  }",
        ]
    W = B // 32
    lines += [
        "  // phase 2: warp butterfly (xor 16, 8, 4, 2, 1); every lane ends with the same value",
        f"  {ct} rs_s = rs_acc;",
        "#pragma unroll",
        f"  for (int rs_o = 16; rs_o > 0; rs_o >>= 1) rs_s = {add('rs_s', shfl)};",
        f"  __shared__ {ct} rs_w[{W}];",
        "  __shared__ bool rs_last;",
        "  __shared__ unsigned rs_ep;",
        "  if ((threadIdx.x & 31) == 0 && threadIdx.x < RS_B) rs_w[threadIdx.x >> 5] = rs_s;",
        "  __syncthreads();",
        "  // phase 3: block butterfly over the warp totals (warp 0)",
        "  if (threadIdx.x < 32) {",
        f"    rs_s = threadIdx.x < {W} ? rs_w[threadIdx.x] : {zero};",
        "#pragma unroll",
        f"    for (int rs_o = 16; rs_o > 0; rs_o >>= 1) rs_s = {add('rs_s', shfl)};",
        "    if (threadIdx.x == 0) {",
        "      // a relaxed ticket (the launch counter never resets: launch L takes tickets",
        "      // [L*G, (L+1)*G), so its epoch is L + 1), then the partial published with",
        "      // its epoch in ONE 64-bit store — no release fence before the ticket, no",
        "      // acquire after it: the last block spins until every slot carries the epoch",
        "      const unsigned long long rs_t = atomicAdd(rs_ticket, 1ull);",
        "      rs_ep = (unsigned)(rs_t / RS_G) + 1u;",
        f"      rs_slot_put(rs_partials + blockIdx.x, rs_ep, {to_bits('rs_s')});",
        "      rs_last = rs_t % RS_G == RS_G - 1;",
        "    }",
        "  }",
        "  __syncthreads();",
        "  if (!rs_last || threadIdx.x >= RS_B) return;",
        "  // phase 4 (last block): thread-strided left folds of the block partials, then butterflies",
        f"  {ct} rs_p = {zero};",
        "  for (int rs_b = threadIdx.x; rs_b < RS_G; rs_b += RS_B) {",
        f"    rs_p = {add('rs_p', from_bits('rs_slot_get(rs_partials + rs_b, rs_ep)'))};",
        "  }",
        "  rs_s = rs_p;",
        "#pragma unroll",
        f"  for (int rs_o = 16; rs_o > 0; rs_o >>= 1) rs_s = {add('rs_s', shfl)};",
        "  if ((threadIdx.x & 31) == 0) rs_w[threadIdx.x >> 5] = rs_s;",
        "  asm volatile(\"bar.sync 1, %0;\" :: \"r\"(RS_B));  // the folding warps only",
        "  if (threadIdx.x < 32) {",
        f"    rs_s = threadIdx.x < {W} ? rs_w[threadIdx.x] : {zero};",
        "#pragma unroll",
        f"    for (int rs_o = 16; rs_o > 0; rs_o >>= 1) rs_s = {add('rs_s', shfl)};",
        "    if (threadIdx.x == 0) {",
        "      // the n % 4 tail terms, in order, after the folded float4 part",
        f"      for (int rs_j = 4 * RS_N4; rs_j < {r(loop.bound)}; ++rs_j) rs_s = {add('rs_s', tail_term)};",
    ]
    if not peers:
        lines += [
        f"      {ct} {acc.name} = {vr_plain(init.value)};",
        f"      {acc.name} = {add(acc.name, 'rs_s')};",
        ]
    else:
        lines += [
            "      // this rank's total (its unit's own result), published to every rank's slot `me`;",
            "      // then the R totals in rank order (every rank computes the same fold)",
            f"      {ct} rs_mine = {vr_plain(init.value)};",
            f"      rs_mine = {add('rs_mine', 'rs_s')};",
            f"      constexpr int RS_R = {peers};",
            "      const unsigned rs_e = ++*rs_epoch;  // this launch's epoch: every rank counts the same launches",
            "      const int rs_me = (int)rs_xtab[RS_R];",
            "      // two slot banks by epoch parity: a rank that has read every epoch-e total may publish",
            "      // e + 1 before a slower rank has read e; it cannot reach e + 2 before that rank",
            "      // has published e + 1, i.e. finished reading e — so no slot is overwritten unread",
            "      const int rs_bank = (int)(rs_e & 1u) * RS_R;",
            "      for (int rs_k = 0; rs_k < RS_R; ++rs_k)",
            "        rs_xchg_put(reinterpret_cast<unsigned long long*>(rs_xtab[rs_k]) + rs_bank + rs_me, rs_e,",
            "                    __float_as_uint(rs_mine));",
            "      const unsigned long long* rs_slots = reinterpret_cast<const unsigned long long*>(rs_xtab[rs_me]) + rs_bank;",
            f"      {ct} {acc.name} = __uint_as_float(rs_xchg_get(rs_slots, rs_e));",
            "      for (int rs_k = 1; rs_k < RS_R; ++rs_k)",
            f"        {acc.name} = {add(acc.name, '__uint_as_float(rs_xchg_get(rs_slots + rs_k, rs_e))')};",
        ]
    for s_ in post:
        lines += [("      " + x) for x in thread_lines(prog, s_, exact)]
    lines += [
        "    }",
        "  }",
        "}",
    ]
    ws_p = f"rs_ws_{base_name}_partials"
    ws_t = f"rs_ws_{base_name}_ticket"
    plan = {
        "name": name,
        "kind": "reduce",
        "grid": G,
        "block": nthreads,
        "smem": smem,
        "pre": pre,
        "fmad": False,
        "order": "reassociated",
        "workspace": [{"name": ws_p, "ctype": "int", "size": str(2 * G)},  # G 64-bit slots
                      {"name": ws_t, "ctype": "int", "size": "2"}],  # one 64-bit counter
        "extra_args": [{"kind": "workspace", "name": ws_p}, {"kind": "workspace", "name": ws_t}],
    }
    if peers:
        ws_e = f"rs_ws_{base_name}_epoch"
        plan["workspace"].append({"name": ws_e, "ctype": "int", "size": "1"})
        plan["extra_args"] += [{"kind": "peer_table"}, {"kind": "workspace", "name": ws_e}]
        plan["peer_ranks"] = peers
        plan["peer_exchange"] = True
    return IdiomKernel(name, "\n".join(lines) + "\n", plan)


def _launch_reduce(st, nats, sm):
    return (st["grid"], 1, 1), (st["block"], 1, 1), st.get("smem", 0), (1, 1, 1)


LAUNCHERS = {
    "rowfold": _launch_rowfold,
    "reduce": _launch_reduce,
    "stencil2d": tmpl_stencil.launch,
    "allpairs": tmpl_allpairs.launch,
    "gemm_tc": tmpl_gemm.launch,
    "seqfold": tmpl_seqfold.launch,
    "iterate": tmpl_iterate.launch,
    "gridseq": tmpl_gridseq.launch,
    "transpose2d": tmpl_transpose.launch,
    "stencil1d": tmpl_stencil1d.launch,
}
