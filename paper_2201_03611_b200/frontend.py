"""The RISE API entry points, exactly as the reference exposes them.

`compile_program` chains the reference's own stages (SURVEY.md §3 call stack
1): parse (parser.py:483) -> infer (typecheck.py:242) -> parse_strategy +
rewrite (strategy.py:329) -> translate_unit (lowering.py:592).  Nothing here
re-implements them; the B200 backend starts at the `ImperativeUnit`.
"""

from __future__ import annotations

from dataclasses import dataclass

from . import extension
from ._ref import errors, lowering, parser, primitives, rules, strategy, typecheck


@dataclass
class Compiled:
    name: str
    source_typed: object  # typed RISE before rewriting
    lowered: object  # typed RISE after the strategy
    unit: object  # lowering.ImperativeUnit
    assumptions: tuple
    free_sizes: tuple


def registry():
    return extension.install(primitives.default_registry())


def typed_program(source: str, assumptions=()):
    reg = registry()
    name, e = parser.parse(source, reg)
    result = typecheck.infer(e, reg, assumptions=list(assumptions)) if assumptions else typecheck.infer(e, reg)
    return name, result.expr, tuple(result.free_sizes)


def rewrite(typed, strategy_text: str):
    reg = registry()
    strat = strategy.parse_strategy(strategy_text, rules.rule_factories(), surface_of=reg.surface_name)
    ctx = strategy.RewriteContext(registry=reg)
    outcome = strat(typed, ctx)
    if isinstance(outcome, strategy.Failure):
        StrategyError = errors.StrategyError

        raise StrategyError(f"strategy failed: {outcome}")
    return outcome.expr, ctx


def compile_program(source: str, strategy_text: str | None = None, name: str | None = None,
                    target: str = "opencl", assumptions=()) -> Compiled:
    """RISE text (+ optional .elv strategy) -> ImperativeUnit."""
    import sys

    # the reference's recursive passes (inference, translation, phrase
    # substitution) nest deeply on larger programs such as nbody
    if sys.getrecursionlimit() < 20000:
        sys.setrecursionlimit(20000)
    pname, typed, free = typed_program(source, assumptions)
    lowered = typed
    asms = list(assumptions)
    if strategy_text:
        lowered, rctx = rewrite(typed, strategy_text)
        asms += [a for a in rctx.assumptions if a not in asms]
        free = tuple(free) + tuple(s for s in rctx.free_sizes if s not in free)
    tctx = lowering.TranslationContext(target=target, assumptions=tuple(asms))
    unit = lowering.translate_unit(lowered, pname or name or "rise", tctx, free_sizes=tuple(free))
    return Compiled(pname or name or "rise", typed, lowered, unit, tuple(asms), tuple(free))
