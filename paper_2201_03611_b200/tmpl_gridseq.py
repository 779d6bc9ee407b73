"""`gridseq` template: a top-level sequential loop that encloses parallel
loops, over the whole GPU instead of one block.

The reference's imperative DPIA allows a sequential `for` (or `ifLess`, or a
plain sequence) whose body contains `parFor`s, e.g. `mapSeq(mapGlobal(f))`
or a fold whose step is a parallel map.  A kernel's blocks cannot wait for
each other, so the generic emission (emit_cuda.GenericKernel.block) runs
such a stage in ONE block — correct, and a performance cliff
(SingleBlockStage).  Here the stage runs on a cooperatively launched grid
(one block per SM, all co-resident; the launch fails instead of hanging when
they are not, RS_LAUNCH_COOPERATIVE):

* every thread follows the sequential control flow (loop bounds and ifLess
  conditions are sizes: uniform across the grid);
* each parallel loop is a grid-stride loop over all threads, followed by a
  grid-wide barrier (`rs_grid_sync`: this loop's writes are what the next
  statement reads);
* a sequential statement with no parallel loop inside runs in global thread
  0, followed by a barrier;
* block-level allocations (the generic kernel's `__shared__` scalars and
  arrays) become global workspaces, visible to every block after a barrier.

Order: PRESERVED — every statement runs once, in the program's order, with
the program's own arithmetic: bit-identical to the generic kernel.  Chosen
when every top-level parallel loop has at least GRIDSEQ_MIN_PAR iterations
(a launch-time precondition; below that the barriers cost more than one
block's serial work, and the single-block kernel runs).
"""

from __future__ import annotations

import os

from . import lir
from ._ref import nat
from .emit_cuda import GenericKernel, NatRenderer, Stage, contains_parfor, kernel_head, py_expr

BLOCK = 512
GRIDSEQ_MIN_PAR = int(os.environ.get("RISE_GRIDSEQ_MIN_PAR", "4096"))


def _top_parfors(s, out):
    """The parallel loops the grid runs (not nested in another parallel loop)."""
    if isinstance(s, lir.ParFor):
        out.append(s)
        return
    if isinstance(s, lir.Seq):
        for c in s.stmts:
            _top_parfors(c, out)
    elif isinstance(s, (lir.For, lir.Alloc)):
        _top_parfors(s.body, out)
    elif isinstance(s, lir.IfLess):
        _top_parfors(s.then, out)
        _top_parfors(s.els, out)


def _block_allocs(s, out):
    """Allocations outside every parallel loop (shared by the whole grid)."""
    if isinstance(s, lir.ParFor) or not contains_parfor(s):
        return
    if isinstance(s, lir.Alloc):
        out.append(s)
        _block_allocs(s.body, out)
    elif isinstance(s, lir.Seq):
        for c in s.stmts:
            _block_allocs(c, out)
    elif isinstance(s, lir.For):
        _block_allocs(s.body, out)
    elif isinstance(s, lir.IfLess):
        _block_allocs(s.then, out)
        _block_allocs(s.els, out)


def _supported(s) -> bool:
    for t in lir.walk(s):
        if isinstance(t, (lir.DoubleBuffer, lir.Raw)):
            return False
    return True


def match(prog, stage, base_name, temps, exact):
    if stage.kind != "block" or not _supported(stage.stmt):
        return None
    pars = []
    _top_parfors(stage.stmt, pars)
    if not pars:
        return None
    allocs = []
    _block_allocs(stage.stmt, allocs)
    name = f"{base_name}_gridseq"
    r = NatRenderer(prog.clamps)
    g = GenericKernel(prog, Stage("serial", stage.stmt), "_", [], exact)
    ws_names = {a.name: f"rs_ws_{base_name}_{a.name}" for a in allocs}
    # (no __restrict__: the workspaces are written and re-read across the grid barriers)
    extra = [f"{a.ctype}* {ws_names[a.name]}" for a in allocs] + ["unsigned* rs_gbar"]
    lines = kernel_head(prog, name, temps, launch_bounds=BLOCK, extra_params=extra)
    lines += [
        "  const int rs_tid = blockIdx.x * blockDim.x + threadIdx.x;",
        "  const int rs_nt = gridDim.x * blockDim.x;",
    ]

    def grid(s, ind):
        p = "  " * ind
        if isinstance(s, lir.Seq):
            out = []
            for c in s.stmts:
                out += grid(c, ind)
            return out
        if not contains_parfor(s):
            return ([f"{p}if (rs_tid == 0) {{"] + g.thread(s, ind + 1)
                    + [f"{p}}}", f"{p}rs_grid_sync(rs_gbar);"])
        if isinstance(s, lir.ParFor):
            return ([f"{p}for (int {s.var} = rs_tid; {s.var} < {r(s.bound)}; {s.var} += rs_nt) {{"]
                    + g.thread(s.body, ind + 1) + [f"{p}}}", f"{p}rs_grid_sync(rs_gbar);"])
        if isinstance(s, lir.Alloc):
            ws = ws_names[s.name]
            decl = (f"{p}{s.ctype}* const {s.name} = {ws};" if s.dims else f"{p}{s.ctype}& {s.name} = *{ws};")
            return [decl] + grid(s.body, ind)
        if isinstance(s, lir.For):
            return ([f"{p}for (int {s.var} = 0; {s.var} < {r(s.bound)}; {s.var} += 1) {{"]
                    + grid(s.body, ind + 1) + [f"{p}}}"])
        if isinstance(s, lir.IfLess):
            return ([f"{p}if ({r(s.lhs)} < {r(s.threshold)}) {{"] + grid(s.then, ind + 1) + [f"{p}}} else {{"]
                    + grid(s.els, ind + 1) + [f"{p}}}"])
        return None

    body = grid(stage.stmt, 1)
    if body is None:
        return None
    lines += body + ["}"]

    def size_of(a):
        n = nat.Const(1)
        for d in a.dims:
            n = n * d
        return py_expr(nat.normalize(n))

    wsb = f"rs_ws_{base_name}_gbar"
    plan = {
        "name": name,
        "kind": "gridseq",
        "block": BLOCK,
        "cooperative": True,
        "fmad": False,
        "order": "preserved",
        "pre": [f"({py_expr(p.bound)}) >= {GRIDSEQ_MIN_PAR}" for p in pars],
        "workspace": [{"name": ws_names[a.name], "ctype": a.ctype, "size": size_of(a)} for a in allocs]
        + [{"name": wsb, "ctype": "int", "size": "2"}],
        "extra_args": [{"kind": "workspace", "name": ws_names[a.name]} for a in allocs]
        + [{"kind": "workspace", "name": wsb}],
    }
    return "\n".join(lines) + "\n", plan


def launch(st, nats, sm):
    # one block per SM: every block of the cooperative launch is resident
    return (max(1, sm), 1, 1), (st["block"], 1, 1), 0, (1, 1, 1)
