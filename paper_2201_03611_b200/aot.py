"""Ahead-of-time nvcc build of the benchmark kernels (build-time check).

The runtime compiles kernel text with NVRTC at run time; this module feeds
the same emitted text for every benchmark config to `nvcc -cubin` for
sm_100a so template errors surface at build time and the cubins can be
disassembled (`cuobjdump -sass`) for the SASS evidence in profiles/.
"""

from __future__ import annotations

import subprocess
from pathlib import Path

from . import programs
from .emit_cuda import emit_cuda, eval_py
from .runtime import INCLUDE_DIR


def _name_exprs(plan, nats):
    targs = ", ".join(str(nats[n]) for n in plan["nat_params"])
    out = []
    for st in plan["stages"]:
        for s in (st, st.get("fallback")):
            if s:
                out.append(f"{s['name']}<{targs}>" if targs else s["name"])
    return out


def build_all(nvcc, arch, out_dir: Path, keys=None):
    out_dir = Path(out_dir)
    out_dir.mkdir(exist_ok=True)
    built = []
    for key in keys or programs.CONFIGS:
        cfg = programs.CONFIGS[key]
        try:
            compiled = programs.compile_config(key)
        except Exception as exc:  # noqa: BLE001 - report, keep building the rest
            print(f"aot: {key}: front end failed: {exc}")
            continue
        code = emit_cuda(compiled.unit)
        nats = dict(cfg["nats"])
        for p in code.plan["nat_params"]:
            nats.setdefault(p, 1)
        for st in code.plan["stages"]:  # sanity: plan expressions evaluate
            eval_py(st.get("total", st.get("rows", "1")), nats)
        refs = ", ".join(f"(void*)&{e}" for e in _name_exprs(code.plan, nats))
        src = out_dir / f"aot_{key}.cu"
        src.write_text(code.text + f"\n__device__ void* rs_aot_refs_{key}[] = {{ {refs} }};\n")
        cubin = out_dir / f"aot_{key}.cubin"
        # the same contraction switch the runtime passes to NVRTC (run.Executable)
        fmad = any(st.get("fmad", False) for st in code.plan["stages"])
        cmd = [nvcc, "-cubin", *arch, "-std=c++17", "-lineinfo", "-O3", f"--fmad={'true' if fmad else 'false'}",
               f"-I{INCLUDE_DIR}", "-o", str(cubin), str(src)]
        print("+", " ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        built.append(cubin)
    return built
