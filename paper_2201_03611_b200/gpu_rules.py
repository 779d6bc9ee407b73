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


def split_reduce(c=None):
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
        partials = Apply(DepApply(Primitive("toMem"), AddressSpace.GLOBAL),
                         Apply(Apply(Primitive("map"), partial), chunks))
        return Apply(Apply(Apply(Primitive("reduce"), op), init), partials)

    return rule(f"splitReduce({nat.to_text(size)})")(matcher)


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


RULES = {
    "splitReduce": split_reduce,
    "splitMap": lambda: split_map,
}
RULE_PARAMS = {
    "splitReduce": "(size: Nat = c)",
    "splitMap": "",
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


def install(rules_module):
    rules_module.RULES.update(RULES)
    rules_module.RULE_PARAMS.update(RULE_PARAMS)


__all__ = ["split_reduce", "split_map", "RULES", "RULE_PARAMS", "CHUNKED_REDUCE_STRATEGY", "install"]
