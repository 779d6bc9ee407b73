"""The reference-side binding of INTEGRATION.md §1, as code: what a `risec`
maintainer adds so that the reference's own entry points reach this back end.

`install()` makes, in the (installed, otherwise unchanged) reference package:

* `codegen.TARGETS` gain "sm100a" and `codegen.emit(unit, "sm100a")`
  returns this back end's text (codegen.py:30, codegen.py:451); every other
  target — and the rejected "cuda" (test_codegen.py:151-154) — behaves as
  before;
* `cli.emit` (the name cli.py:16 imported) and the CLI's `--target` choices
  (cli.py:245) follow, so `risec prog.rise --target sm100a` emits sm_100a
  CUDA;
* `cexec.run_emitted(code, unit, nats, inputs)` (cexec.py:555) runs text
  this back end emitted on the GPU through `run_cuda` (same argument order,
  same nested result), and any other text through the reference's own
  evaluator.

Idempotent; `uninstall()` restores the reference's functions.
"""

from __future__ import annotations

from ._ref import cexec, cli, codegen
from .emit_cuda import TARGET

HEADER = "// rise-b200 sm100a"

_saved: dict = {}


def _emit(unit, target):
    if target == TARGET:
        from .emit_cuda import emit_cuda

        return emit_cuda(unit).text
    return _saved["emit"](unit, target)


def _run_emitted(code, unit, nat_assignment, inputs):
    if isinstance(code, str) and code.startswith(HEADER):
        from .run import run_cuda

        return run_cuda(code, unit, nat_assignment, inputs)
    return _saved["run_emitted"](code, unit, nat_assignment, inputs)


def _build_arg_parser():
    ap = _saved["build_arg_parser"]()
    for action in ap._actions:  # argparse keeps choices on the action
        if "--target" in action.option_strings and TARGET not in action.choices:
            action.choices = tuple(action.choices) + (TARGET,)
    return ap


def install():
    if _saved:
        return
    _saved.update(emit=codegen.emit, targets=codegen.TARGETS, cli_emit=cli.emit,
                  run_emitted=cexec.run_emitted, build_arg_parser=cli.build_arg_parser)
    codegen.TARGETS = tuple(codegen.TARGETS) + (TARGET,)
    codegen.emit = _emit
    cli.emit = _emit
    cli.build_arg_parser = _build_arg_parser
    cexec.run_emitted = _run_emitted


def uninstall():
    if not _saved:
        return
    codegen.emit = _saved["emit"]
    codegen.TARGETS = _saved["targets"]
    cli.emit = _saved["cli_emit"]
    cli.build_arg_parser = _saved["build_arg_parser"]
    cexec.run_emitted = _saved["run_emitted"]
    _saved.clear()
