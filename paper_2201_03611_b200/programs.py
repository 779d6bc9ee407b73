"""The benchmark programs, written against the reference's RISE API.

Each config of BASELINE.json is a RISE program (plus an Elevate strategy
where the program is still high-level) that goes through the unchanged
front end (`frontend.compile_program`) and then the sm100a back end.

* C1 `dot`   — map(*) + reduce(+), lowered by `fuseReduceMap ; toReduceSeq`
               (BASELINE.md §4 row C1).
* C2 `mv`    — the paper's matrix-vector program (Listing 1; the
               reference's tests/data/mv.rise) with either the
               `toMapGlobal` strategy or the paper's
               Listing-3 strategy (tests/data/mv_opt.elv).
* C3 `conv`  — 3x3 stencil: padClamp2D + slide2D + map/reduce (SURVEY.md
               §8.1 validated form), weights as an Array[3, Array[3, f32]].
* C4 `sgemm` — A x B with B given transposed (`Bt`), the form the reference
               can already translate and emit (SURVEY.md §8 c, C4); and
               `sgemm_tiled`, the tiled split / transpose / toMem(Local)
               lowering BASELINE.json names.
* C5 `nbody` — all-pairs accelerations + Euler velocity update (one step),
               positions Array[n, Array[3, f32]] and masses Array[n, f32].
"""

from __future__ import annotations

DOT = """\
depFun((n: Nat) => fun(a: Array[n, f32] => fun(b: Array[n, f32] =>
  zip(a)(b) |> map(fun(p => fst(p) * snd(p))) |> reduce(add)(0.0f) )))
"""
DOT_STRATEGY = "fuseReduceMap @ every(isReduce) ; toReduceSeq @ every(isReduce)"

# the north star's other memory-bound reduction: asum = sum |x_i| (needs the
# extension's `abs`)
ASUM = """\
depFun((n: Nat) => fun(x: Array[n, f32] => x |> map(fun(v => abs(v))) |> reduce(add)(0.0f) ))
"""
ASUM_STRATEGY = DOT_STRATEGY

# C1 written in an explicit, parallel order: 4096-element chunks folded
# left-to-right in parallel (one row per thread, the `rowfold` template),
# then the chunk partials folded left-to-right.  Emitted with
# reassociate=False every step keeps this order: bit-exact with the
# reference.  Needs the divisibility assumption 4096 | n.
DOT_CHUNKED = """\
depFun((n: Nat) => fun(a: Array[n, f32] => fun(b: Array[n, f32] =>
  zip(a)(b) |> split(4096)
    |> mapGlobal(fun(ch => ch |> reduceSeq(Private)(fun(acc, p => acc + fst(p) * snd(p)))(0.0f)))
    |> toMem(Global)
    |> reduceSeq(Private)(fun(acc, v => acc + v))(0.0f) )))
"""
DOT_CHUNK = 4096
# ... and the same schedule derived from DOT by the GPU rewrite rules
from .gpu_rules import CHUNKED_REDUCE_STRATEGY as DOT_CHUNKED_STRATEGY  # noqa: E402

MV = """\
// matrix-vector multiplication: for each row, a dot product with x
def mv = depFun((n: Nat, m: Nat) =>
  fun(M: Array[n, Array[m, f32]] =>
    fun(x: Array[m, f32] =>
      M |> map(fun(row =>
          zip(row)(x) |>
            map(fun(ax => fst(ax) * snd(ax))) |>
              reduce(add)(0.0f) )) )) )
"""
MV_GLOBAL_STRATEGY = (
    "toMapGlobal @ outermost(isMap) ; fuseReduceMap @ every(isReduce) ; toReduceSeq @ every(isReduce)"
)
# the paper's Listing 3
MV_OPT_STRATEGY = """\
    splitJoinMap    `@` outermost(isMap)    `;`
    toMapWorkGroup  `@` outermost(isMap)    `;`
    toMapLocal      `@` outermost(isMap)    `;`
    fuseReduceMap   `@` every(isReduce)     `;`
    toReduceSeq     `@` every(isReduce)
"""

CONV = """\
def conv = depFun((n: Nat, m: Nat) => fun(img: Array[n, Array[m, f32]] => fun(w: Array[3, Array[3, f32]] =>
  img |> padClamp2D(1)(1) |> slide2D(3)(1) |> mapGlobal(mapGlobal(fun(win =>
    zip(win)(w)
      |> mapSeq(fun(rw => zip(fst(rw))(snd(rw)) |> reduceSeq(Private)(fun(acc, p => acc + fst(p) * snd(p)))(0.0f)))
      |> toMem(Private)
      |> reduceSeq(Private)(fun(acc, v => acc + v))(0.0f) ))) )))
"""

SGEMM_BT = """\
def sgemm = depFun((n: Nat, m: Nat, k: Nat) =>
  fun(A: Array[n, Array[k, f32]] => fun(Bt: Array[m, Array[k, f32]] =>
    A |> mapGlobal(fun(arow => Bt |> mapGlobal(fun(brow =>
      zip(arow)(brow) |> reduceSeq(Private)(fun(acc, p => acc + fst(p) * snd(p)))(0.0f) ))) ))))
"""

NBODY = """\
def nbody = depFun((n: Nat) =>
  fun(pos: Array[n, Array[3, f32]] => fun(vel: Array[n, Array[3, f32]] => fun(mass: Array[n, f32] =>
    zip(pos)(vel) |> mapGlobal(fun(pv =>
      zip(transpose(pos))(zip(fst(pv))(snd(pv))) |> mapSeq(fun(col =>
        snd(snd(col)) + 0.01f *
          (zip(fst(col))(zip(pos)(mass)) |> reduceSeq(Private)(fun(acc, q =>
             acc + (fst(q) - fst(snd(col))) *
               (snd(snd(q)) *
                 ((zip(fst(snd(q)))(fst(pv)) |> reduceSeq(Private)(fun(r2, d => r2 + (fst(d) - snd(d)) * (fst(d) - snd(d))))(0.01f))
                   |> fun(r2 => rsqrt(r2) * rsqrt(r2) * rsqrt(r2)))) ))(0.0f)) )) )) ))))
"""

# C4 without the pre-transposed operand: B is K x N row-major, read through
# the extension's transpose (the tensor-core template takes it MN-major)
SGEMM = """\
def sgemm = depFun((n: Nat, m: Nat, k: Nat) =>
  fun(A: Array[n, Array[k, f32]] => fun(B: Array[k, Array[m, f32]] =>
    A |> mapGlobal(fun(arow => transpose(B) |> mapGlobal(fun(bcol =>
      zip(arow)(bcol) |> reduceSeq(Private)(fun(acc, p => acc + fst(p) * snd(p)))(0.0f) ))) ))))
"""

# C4 as BASELINE.json names it: the tiled lowering.  Work-groups take row
# blocks of A (split(2)); each stages its block in Local memory (toMem(Local),
# the work-items copying each row together); the work-items then
# walk the columns of B (read through transpose: B is row-major K x N), and
# each output is folded over K in tiles of 32 (split(32)): per-tile partial
# dot products, then their sum.  Needs 2 | n and 32 | k (SGEMM_TILED_ASSUMPTIONS).
# The generic kernel runs it in exactly this order (bit-exact with the
# reference semantics); the gemm_tc template recognises the same contraction
# through the staging and the K tiles (tmpl_gemm.match_tiled) and runs it on
# the tensor cores (3xTF32, fp64 error bound).
SGEMM_TILED = """\
def sgemmTiled = depFun((n: Nat, m: Nat, k: Nat) =>
  fun(A: Array[n, Array[k, f32]] => fun(B: Array[k, Array[m, f32]] =>
    A |> split(2) |> mapWorkGroup(fun(aBlock =>
      aBlock |> mapSeq(mapLocal(fun(v => v * 1.0f))) |> toMem(Local)
        |> mapSeq(fun(arow =>
          transpose(B) |> mapLocal(fun(bcol =>
            zip(arow)(bcol) |> split(32)
              |> mapSeq(fun(tile => tile |> reduceSeq(Private)(fun(acc, p => acc + fst(p) * snd(p)))(0.0f)))
              |> toMem(Private)
              |> reduceSeq(Private)(fun(acc, v => acc + v))(0.0f) )) )) )) |> join )))
"""
SGEMM_TILE_ROWS, SGEMM_TILE_K = 2, 32

# the high-level programs the GPU strategies (gpu_rules.*_STRATEGY) lower to
# CONV, SGEMM_TILED and NBODY (SURVEY.md §8 f 3)
CONV_HIGH = """\
def conv = depFun((n: Nat, m: Nat) => fun(img: Array[n, Array[m, f32]] => fun(w: Array[3, Array[3, f32]] =>
  img |> padClamp2D(1)(1) |> slide2D(3)(1) |> map(map(fun(win =>
    zip(win)(w)
      |> map(fun(rw => zip(fst(rw))(snd(rw)) |> map(fun(p => fst(p) * snd(p))) |> reduce(add)(0.0f)))
      |> reduce(add)(0.0f) ))) )))
"""

SGEMM_HIGH = """\
def sgemmTiled = depFun((n: Nat, m: Nat, k: Nat) =>
  fun(A: Array[n, Array[k, f32]] => fun(B: Array[k, Array[m, f32]] =>
    A |> map(fun(arow => transpose(B) |> map(fun(bcol =>
      zip(arow)(bcol) |> map(fun(p => fst(p) * snd(p))) |> reduce(add)(0.0f) )))) )))
"""

NBODY_HIGH = """\
def nbody = depFun((n: Nat) =>
  fun(pos: Array[n, Array[3, f32]] => fun(vel: Array[n, Array[3, f32]] => fun(mass: Array[n, f32] =>
    zip(pos)(vel) |> map(fun(pv =>
      zip(transpose(pos))(zip(fst(pv))(snd(pv))) |> map(fun(col =>
        snd(snd(col)) + 0.01f *
          (zip(fst(col))(zip(pos)(mass)) |> map(fun(q =>
             (fst(q) - fst(snd(col))) *
               (snd(snd(q)) *
                 ((zip(fst(snd(q)))(fst(pv)) |> map(fun(d => (fst(d) - snd(d)) * (fst(d) - snd(d)))) |> reduce(add)(0.01f))
                   |> fun(r2 => rsqrt(r2) * rsqrt(r2) * rsqrt(r2)))) )) |> reduce(add)(0.0f)) )) )) ))))
"""


def sgemm_tiled_assumptions():
    from ._ref import nat

    return ((nat.Var("n"), nat.Const(SGEMM_TILE_ROWS)), (nat.Var("k"), nat.Const(SGEMM_TILE_K)))


# the same step for a block of t target bodies against all n sources (the
# per-GPU program of the multi-GPU decomposition, shard.sharded_nbody)
NBODY_SHARD = """\
def nbodyShard = depFun((t: Nat, n: Nat) =>
  fun(tpos: Array[t, Array[3, f32]] => fun(tvel: Array[t, Array[3, f32]] =>
  fun(pos: Array[n, Array[3, f32]] => fun(mass: Array[n, f32] =>
    zip(tpos)(tvel) |> mapGlobal(fun(pv =>
      zip(transpose(pos))(zip(fst(pv))(snd(pv))) |> mapSeq(fun(col =>
        snd(snd(col)) + 0.01f *
          (zip(fst(col))(zip(pos)(mass)) |> reduceSeq(Private)(fun(acc, q =>
             acc + (fst(q) - fst(snd(col))) *
               (snd(snd(q)) *
                 ((zip(fst(snd(q)))(fst(pv)) |> reduceSeq(Private)(fun(r2, d => r2 + (fst(d) - snd(d)) * (fst(d) - snd(d))))(0.01f))
                   |> fun(r2 => rsqrt(r2) * rsqrt(r2) * rsqrt(r2)))) ))(0.0f)) )) )) )))))
"""

CONFIGS = {
    "dot": dict(source=DOT, strategy=DOT_STRATEGY, name="dot", nats={"n": 1 << 24}),
    "gemv": dict(source=MV, strategy=MV_GLOBAL_STRATEGY, name="mv", nats={"n": 8192, "m": 8192}),
    "gemv_opt": dict(source=MV, strategy=MV_OPT_STRATEGY, name="mv", nats={"n": 8192, "m": 8192, "s": 32}),
    "conv": dict(source=CONV, strategy=None, name="conv", nats={"n": 8192, "m": 8192}),
    "sgemm": dict(source=SGEMM_BT, strategy=None, name="sgemm", nats={"n": 4096, "m": 4096, "k": 4096}),
    "nbody": dict(source=NBODY, strategy=None, name="nbody", nats={"n": 131072}),
    "sgemm_tiled": dict(source=SGEMM_TILED, strategy=None, name="sgemmTiled",
                        nats={"n": 4096, "m": 4096, "k": 4096}, assumptions=sgemm_tiled_assumptions),
}


def compile_config(key: str):
    from .frontend import compile_program

    cfg = CONFIGS[key]
    asm = cfg.get("assumptions")
    return compile_program(cfg["source"], cfg["strategy"], name=cfg["name"], assumptions=asm() if asm else ())
