"""GPU-oriented rewrite rules in the style of the reference's rule library
(rules.py:47-235), registered in `rules.RULES` / `RULE_PARAMS` (the table
strategy files name rules from, rules.py:237-259) by extension.install().

With them the chunked, two-kernel form of a reduction — the bit-exact GPU
schedule of C1 — is derived from the plain program by a strategy instead
of being written by hand (SURVEY.md §8 f 3):

    DOT |> splitReduce(4096) ; splitMap ; mapFusion ; fuseReduceMap ;
           toMapGlobal ; toReduceSeq          ==  programs.DOT_CHUNKED

Rules, each matching the maximal application chain it is pointed at and
returning an untyped replacement that the strategy engine re-types:

* `splitReduce(c)`: reduce(add)(0)(xs)  ->
      reduce(add)(0)(toMem(Global)(map(reduce(add)(0))(split(c)(xs))))
  Only for `add` with a zero literal init (its identity): the partial
  folds start from the identity, so the rewrite only reassociates the sum
  into c-element chunks.  The partials are materialised in Global memory —
  the two folds become two kernels.  Divisibility of the length by c is
  recorded as an assumption (as splitJoinMap does, rules.py:75-79).
* `splitMap`: split(c)(map(f)(xs))  ->  map(map(f))(split(c)(xs))
  (the map/split commutation that lets a chunk fold fuse with the map that
  feeds it).
* `splitReduce(c, Private)`: the same split with the partials in Private
  memory — K tiles of one work-item's fold (C4).
* `insertToMemReduce(a)`: reduce(op)(init)(map-produced xs)  ->
  reduce(op)(init)(toMem(a)(xs)) — the reduce-consumer dual of the
  reference's insertToMem (C3's row sums before their sum).
* `stageToMem(a)`: map(map(F))(xs)  ->  map(blk => map(F)(toMem(a)(copy
  blk)))(xs) — each block copied into Local memory once (C4's A tiles).

The strategies at the end of this module take the high-level conv, sgemm
and nbody programs (programs.*_HIGH) to exactly the hand-lowered programs
the templates claim (CONV, SGEMM_TILED, NBODY): the emitted sm100a text is
byte-identical (tests/test_emit.py).
"""

from __future__ import annotations

from ._ref import expr as _expr
from ._ref import nat
from ._ref import strategy as _strategy
from ._ref import types as _types

Apply, DepApply, Literal, Primitive, spine = _expr.Apply, _expr.DepApply, _expr.Literal, _expr.Primitive, _expr.spine
Failure, rule = _strategy.Failure, _strategy.rule
AddressSpace = _types.AddressSpace


def _chain(e, tag):
    head, args = spine(e)
    if not isinstance(head, Primitive) or head.name != tag:
        return None
    return head, args


def _apps(args):
    return [a for k, a in args if k == "app"]


def _is_zero(e):
    if not isinstance(e, Literal):
        return False
    text = e.text.strip()
    try:
        return float(e.value) == 0.0 and not text.startswith("-")
    except (TypeError, ValueError):
        return False


def _reduce_length(head):
    """Array length of an instantiated reduce: (op) -> init -> Array[n, t] -> t."""
    t = head.type
    try:
        arr = t.out.out.inp
        return arr.size
    except AttributeError:
        return None


def split_reduce(c=None, a=AddressSpace.GLOBAL):
    """`a` is where the partials live: Global (two kernels, C1's chunked
    schedule) or Private (K tiles inside one work-item, C4's tiled fold)."""
    size = nat.Var("c") if c is None else c
    if isinstance(size, int):
        size = nat.Const(size)

    def matcher(e, ctx):
        m = _chain(e, "reduce")
        if m is None:
            return Failure("not a reduce")
        head, args = m
        apps = _apps(args)
        if len(apps) != 3:
            return Failure("reduce is not saturated")
        op, init, xs = apps
        if not (isinstance(op, Primitive) and op.name == "add"):
            return Failure("splitReduce needs the add primitive (associative with a known identity)")
        if not _is_zero(init):
            return Failure("splitReduce needs the zero literal as init (add's identity)")
        length = _reduce_length(head)
        if length is None:
            return Failure("reduce chain is untyped")
        sn, ln = nat.normalize(size), nat.normalize(length)
        if isinstance(sn, nat.Const) and isinstance(ln, nat.Const):
            if ln.value % sn.value:
                return Failure(f"chunk size {sn.value} does not divide {ln.value}")
        else:
            ctx.assume_divides(size, length)
        if isinstance(size, nat.Var):
            ctx.add_free_size(size.name)
        partial = Apply(Apply(Primitive("reduce"), op), init)
        chunks = Apply(DepApply(Primitive("split"), size), xs)
        partials = Apply(DepApply(Primitive("toMem"), a), Apply(Apply(Primitive("map"), partial), chunks))
        return Apply(Apply(Apply(Primitive("reduce"), op), init), partials)

    return rule(f"splitReduce({nat.to_text(size)}, {a})")(matcher)


@rule("splitMap")
def split_map(e, ctx):
    m = _chain(e, "split")
    if m is None:
        return Failure("not a split")
    _head, args = m
    deps = [a for k, a in args if k == "dep"]
    apps = _apps(args)
    if len(deps) != 1 or len(apps) != 1:
        return Failure("split is not applied to an array")
    inner = _chain(apps[0], "map")
    if inner is None:
        return Failure("split does not consume a map")
    iapps = _apps(inner[1])
    if len(iapps) != 2:
        return Failure("map is not saturated")
    f, xs = iapps
    return Apply(Apply(Primitive("map"), Apply(Primitive("map"), f)), Apply(DepApply(Primitive("split"), deps[0]), xs))


_MAPS = ("map", "mapSeq", "mapGlobal", "mapWorkGroup", "mapLocal")


def insert_to_mem_reduce(a=AddressSpace.PRIVATE):
    """reduce(op)(init)(producer)  ->  reduce(op)(init)(toMem(a)(producer))

    The reduce-consumer dual of the reference's insertToMem (rules.py:207,
    which only fires under map-like consumers): the produced array is
    materialised before it is folded, so the fold stays a separate loop
    (e.g. conv's row sums, then their sum — SURVEY.md §8.1)."""

    def matcher(e, ctx):
        m = _chain(e, "reduce") or _chain(e, "reduceSeq")
        if m is None:
            return Failure("not a reduce")
        head, args = m
        apps = _apps(args)
        if len(apps) != 3:
            return Failure("reduce is not saturated")
        producer = apps[2]
        ptag = _expr.head_primitive(producer)
        if ptag == "toMem":
            return Failure("already materialized")
        if ptag not in _MAPS:
            return Failure("the folded array is not produced by a map")
        out = head
        for k, arg in args[:-1]:
            out = Apply(out, arg) if k == "app" else DepApply(out, arg)
        return Apply(out, Apply(DepApply(Primitive("toMem"), a), producer))

    return rule(f"insertToMemReduce({a})")(matcher)


def _rows_copy():
    """map(map(fun(v => v * 1.0f))): an exact element copy (x * 1 is x for
    every binary32 value, -0.0 and NaN included; x + 0.0f is not)."""
    v = _expr.Identifier("v")
    one = Literal("1.0f", 1.0)
    copy = _expr.Lambda(v, Apply(Apply(Primitive("mul"), v), one))
    return Apply(Primitive("map"), Apply(Primitive("map"), copy))


def stage_to_mem(a=AddressSpace.LOCAL):
    """map(map(F))(xs)  ->  map(fun(blk => map(F)(toMem(a)(copy(blk)))))(xs)

    Every block of a blocked map (e.g. the row blocks splitJoinMap made)
    is copied into `a` memory once, and the inner map reads the copy: the
    Lift/Shine `toLocal` staging of a work-group's tile (SURVEY.md §8 f 3).
    The copy is row by row, element by element (two maps the lowering rules
    then assign: mapSeq over rows, mapLocal over a row's elements)."""

    def matcher(e, ctx):
        m = _chain(e, "map")
        if m is None:
            return Failure("not a map")
        head, args = m
        apps = _apps(args)
        if len(apps) not in (1, 2):
            return Failure("map is not applied to a function")
        inner = _chain(apps[0], "map")
        if inner is None or len(_apps(inner[1])) != 1:
            return Failure("the mapped function is not a map over each block")
        t = head.type
        try:
            blk = t.out.inp.elem  # (s -> t) -> Array[n, s] -> ...: s = one block
            ok = isinstance(blk, _types.ArrayType) and isinstance(blk.elem, _types.ArrayType) and \
                isinstance(blk.elem.elem, _types.ScalarType)
        except AttributeError:
            ok = False
        if not ok:
            return Failure("stageToMem copies blocks of scalar rows (Array[r, Array[c, scalar]])")
        b = _expr.Identifier("blk")
        staged = Apply(DepApply(Primitive("toMem"), a), Apply(_rows_copy(), b))
        body = _expr.Lambda(b, Apply(apps[0], staged))
        out = Apply(Primitive("map"), body)
        return Apply(out, apps[1]) if len(apps) == 2 else out

    return rule(f"stageToMem({a})")(matcher)


RULES = {
    "splitReduce": split_reduce,
    "splitMap": lambda: split_map,
    "insertToMemReduce": insert_to_mem_reduce,
    "stageToMem": stage_to_mem,
}
RULE_PARAMS = {
    "splitReduce": "(size: Nat = c, a: AddrSp = Global)",
    "splitMap": "",
    "insertToMemReduce": "(a: AddrSp = Private)",
    "stageToMem": "(a: AddrSp = Local)",
}

# the bit-exact chunked GPU schedule of a sum, from the plain program
CHUNKED_REDUCE_STRATEGY = """\
    splitReduce(4096)     `@` outermost(isReduce)        `;`
    splitMap              `@` every(isPrimitive(split))  `;`
    mapFusion             `@` outermost(isMap)           `;`
    try(fuseReduceMap)    `@` every(isReduce)            `;`
    toMapGlobal           `@` outermost(isMap)           `;`
    toReduceSeq           `@` every(isReduce)
"""


# C3: the high-level 3x3 stencil (programs.CONV_HIGH) -> programs.CONV: the
# row sums materialised before their sum, each row's products fused into its
# fold, both folds sequential, the two window maps on the grid, the row map
# sequential
CONV_STRATEGY = """\
    insertToMemReduce(Private)  `@` outermost(isReduce)  `;`
    try(fuseReduceMap)          `@` every(isReduce)      `;`
    toReduceSeq                 `@` every(isReduce)      `;`
    toMapGlobal                 `@` outermost(isMap)     `;`
    toMapGlobal                 `@` outermost(isMap)     `;`
    toMapSeq                    `@` outermost(isMap)
"""

# C4: the high-level product (programs.SGEMM_HIGH) -> programs.SGEMM_TILED:
# rows of A in blocks of 2 per work-group, each block staged in Local
# memory, the columns over the work-items, K folded in tiles of 32
# (per-tile partials in Private memory, then their sum)
SGEMM_TILED_STRATEGY = """\
    splitJoinMap(2)             `@` outermost(isMap)             `;`
    splitReduce(32, Private)    `@` every(isReduce)              `;`
    try(splitMap)               `@` every(isPrimitive(split))    `;`
    try(mapFusion)              `@` every(isMap)                 `;`
    try(fuseReduceMap)          `@` every(isReduce)              `;`
    stageToMem(Local)           `@` outermost(isMap)             `;`
    toReduceSeq                 `@` every(isReduce)              `;`
    toMapWorkGroup              `@` outermost(isMap)             `;`
    toMapSeq                    `@` outermost(isMap)             `;`
    toMapLocal                  `@` outermost(isMap)             `;`
    toMapSeq                    `@` outermost(isMap)             `;`
    toMapSeq                    `@` outermost(isMap)             `;`
    toMapLocal                  `@` outermost(isMap)
"""

# C5: the high-level all-pairs step (programs.NBODY_HIGH) -> programs.NBODY:
# every map/reduce pair fused into a sequential fold, the bodies on the grid,
# the three components sequential
NBODY_STRATEGY = """\
    fuseReduceMap               `@` every(isReduce)      `;`
    toReduceSeq                 `@` every(isReduce)      `;`
    toMapGlobal                 `@` outermost(isMap)     `;`
    toMapSeq                    `@` outermost(isMap)
"""


def install(rules_module):
    rules_module.RULES.update(RULES)
    rules_module.RULE_PARAMS.update(RULE_PARAMS)


__all__ = ["split_reduce", "split_map", "insert_to_mem_reduce", "stage_to_mem", "RULES", "RULE_PARAMS",
           "CHUNKED_REDUCE_STRATEGY", "CONV_STRATEGY", "SGEMM_TILED_STRATEGY", "NBODY_STRATEGY", "install"]
