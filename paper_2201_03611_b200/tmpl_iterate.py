"""`iterate` template: `newDoubleBuffer` over the whole GPU.

Matches the stage the reference's `iterate(k)` lowers to (lowering.py:459-517;
Listing 11 of the paper, codegen.emit_double_buffer, codegen.py:469-504):

    DoubleBuffer(input, output, size):
      for i < k:
        parFor g < bound(i):  body(g) reading in_ptr, writing out_ptr
        ifLess(i < k - 2) swap(in_ptr, out_ptr, flag) else done(out_ptr = output)

The generic emission runs the whole nest in ONE block with the buffers in
shared memory, which caps the problem at a few KiB.  Here the two buffers
are global workspaces, each step's parallel loop is a grid-stride loop over
every thread of a cooperatively launched grid (one block per SM: all
co-resident), consecutive steps are separated by a grid-wide barrier
(`rs_grid_sync`), and the pointer swap runs in every thread on private
copies of in_ptr / out_ptr / flag (it is the same deterministic update
everywhere, so no shared state is needed).

Order: PRESERVED — each output cell of each step is computed by the
program's own body; steps run in order.  Bit-identical to the reference.
"""

from __future__ import annotations

from . import lir
from ._ref import nat
from .emit_cuda import GenericKernel, NatRenderer, Stage, kernel_head, py_expr

BLOCK = 256


def _shape(stage):
    s = stage.stmt
    if not isinstance(s, lir.DoubleBuffer):
        return None
    loop = s.body
    if not isinstance(loop, lir.For):
        return None
    body = loop.body.stmts if isinstance(loop.body, lir.Seq) else [loop.body]
    if len(body) != 2 or not isinstance(body[0], lir.ParFor) or not isinstance(body[1], lir.IfLess):
        return None
    par, sw = body
    # a flat parallel step: no nested parallel loops, no Local / Global allocations
    for t in lir.walk(par.body):
        if isinstance(t, (lir.ParFor, lir.DoubleBuffer)):
            return None
        if isinstance(t, lir.Alloc) and t.space != "Private":
            return None
    if not (isinstance(sw.then, lir.Raw) and isinstance(sw.els, lir.Raw)):
        return None
    return s, loop, par, sw


def match(prog, stage, base_name, temps, exact):
    if stage.kind != "block":
        return None
    shape = _shape(stage)
    if shape is None:
        return None
    db, loop, par, sw = shape
    name = f"{base_name}_iterate"
    r = NatRenderer(prog.clamps)
    c = db.ctype
    g = GenericKernel(prog, Stage("serial", par.body), "_", [], exact)
    body_lines = g.thread(par.body, 3)
    # no __restrict__ on the ping-pong buffers: they are written and re-read
    # across steps (no read-only-cache loads of data other blocks rewrite)
    extra = [f"{c}* buffer1", f"{c}* buffer2", "unsigned* rs_gbar"]
    lines = kernel_head(prog, name, temps, launch_bounds=BLOCK, extra_params=extra)
    lines += [
        f"  const {c}* in_ptr = {db.input_buf};",
        f"  {c}* out_ptr = buffer1;",
        "  unsigned char flag = 1;",
        f"  for (int {loop.var} = 0; {loop.var} < {r(loop.bound)}; {loop.var} += 1) {{",
        f"    for (int {par.var} = blockIdx.x * blockDim.x + threadIdx.x; {par.var} < {r(par.bound)}; "
        f"{par.var} += gridDim.x * blockDim.x) {{",
    ]
    lines += body_lines
    lines += [
        "    }",
        "    rs_grid_sync(rs_gbar);  // this step's writes are the next step's reads",
        f"    if ({r(sw.lhs)} < {r(sw.threshold)}) {{",
    ]
    lines += ["      " + x for x in sw.then.lines]
    lines += ["    } else {"]
    lines += ["      " + x for x in sw.els.lines]
    lines += ["    }", "  }", "}"]
    ws1, ws2, wsb = (f"rs_ws_{base_name}_buf1", f"rs_ws_{base_name}_buf2", f"rs_ws_{base_name}_gbar")
    size = py_expr(nat.normalize(db.size))
    plan = {
        "name": name,
        "kind": "iterate",
        "block": BLOCK,
        "cooperative": True,
        "fmad": False,
        "order": "preserved",
        "pre": [],
        "workspace": [{"name": ws1, "ctype": c, "size": size}, {"name": ws2, "ctype": c, "size": size},
                      {"name": wsb, "ctype": "int", "size": "2"}],
        "extra_args": [{"kind": "workspace", "name": ws1}, {"kind": "workspace", "name": ws2},
                       {"kind": "workspace", "name": wsb}],
    }
    return "\n".join(lines) + "\n", plan


def launch(st, nats, sm):
    # one block per SM: every block of the cooperative launch is resident
    return (max(1, sm), 1, 1), (st["block"], 1, 1), 0, (1, 1, 1)
