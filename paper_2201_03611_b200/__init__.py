"""rise-b200: a B200-native (sm_100a) execution backend for RISE/Shine.

Programs are written against the reference's RISE API (the `risec` front
end, installed in baseline/_ref); this package replaces only the final stage
— imperative DPIA -> kernel -> execution — with hand-written sm_100a kernel
templates, NVRTC, and a native C-ABI runtime (include/rise_b200.h).

Public API (mirrors the reference's back-end entry points):

* `emit(unit, "sm100a")`            — codegen.emit counterpart (codegen.py:451)
* `emit_cuda(unit)`                 — text + launch plan
* `run_cuda(code, unit, nats, ins)` — cexec.run_emitted counterpart (cexec.py:555)
* `Executable(code, nats)`          — compiled, allocation-free launches
* `compile_program(src, strategy)`  — the unchanged RISE front end
"""

from . import extension as _extension
from .emit_cuda import TARGET, CudaCode, emit, emit_cuda, plan_of
from .frontend import compile_program, registry
from .run import Executable, executable, run_cuda

_extension.install()

__all__ = [
    "TARGET",
    "CudaCode",
    "Executable",
    "compile_program",
    "emit",
    "emit_cuda",
    "executable",
    "plan_of",
    "registry",
    "run_cuda",
]
