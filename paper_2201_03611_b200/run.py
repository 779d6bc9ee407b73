"""Execution of emitted sm100a kernel text: the CUDA counterpart of
`cexec.run_emitted` / `cexec.execute_kernel` (cexec.py:509-581).

`run_cuda(code, unit, nat_assignment, inputs)` keeps run_emitted's argument
order and result form (nested lists of np.float32 / int, the interpreter's
value form), so oracle comparisons read exactly like the reference's own
tests (test_codegen.py:157-183).  `Executable` is the allocation-free path
used by benchmarks: compiled once per (text, sizes), launched on device
buffers (any object exposing `data_ptr()`, e.g. torch CUDA tensors, or raw
integer device pointers).

Every launch goes through the native runtime (`runtime.Function.launch` ->
rs_launch).  There is no CPU fallback: without the runtime library or a GPU
this module raises.
"""

from __future__ import annotations

import ctypes
import math
import threading

import numpy as np

from . import runtime as rt
from ._ref import errors, interpreter, nat
from ._ref import types as _types
from .emit_cuda import CudaCode, eval_py, plan_of

InterpreterError = errors.InterpreterError
ArrayType, ScalarType = _types.ArrayType, _types.ScalarType

INT32_MAX = 2**31 - 1


def _launchers():
    from . import idioms

    return idioms.LAUNCHERS


class Executable:
    """Kernel text specialised to concrete sizes, compiled and loaded."""

    def __init__(self, code, nats: dict, device: int | None = None):
        text = code.text if isinstance(code, CudaCode) else code
        self.text = text
        self.plan = plan_of(text)
        self.nats = {}
        for name in self.plan["nat_params"]:
            if name not in nats:
                raise InterpreterError(f"missing size argument {name!r}")
            self.nats[name] = int(nats[name])
        rt.init(device)
        self.sm_count = rt.device_attribute(rt.SM_COUNT_ATTR)
        self.output_size = eval_py(self.plan["output"]["size"], self.nats)
        self.input_sizes = {
            i["name"]: (None if i["scalar"] else eval_py(i["size"], self.nats)) for i in self.plan["inputs"]
        }
        self.temp_sizes = {t["name"]: eval_py(t["size"], self.nats) for t in self.plan["temps"]}
        for what, size in [("output", self.output_size)] + list(self.input_sizes.items()) + list(
            self.temp_sizes.items()
        ):
            if size is not None and size > INT32_MAX:
                raise InterpreterError(f"{what} has {size} elements; 32-bit indexing supports < 2^31")
        targs = ", ".join(str(self.nats[n]) for n in self.plan["nat_params"])
        self.launches = []
        exprs = []
        fmad = False
        for st in self.plan["stages"]:
            chosen = st
            if st.get("pre") and not all(eval_py(p, self.nats) for p in st["pre"]):
                if st.get("peer_ranks") or st.get("peer_halo") or st.get("peer_out"):
                    raise InterpreterError(f"{st['name']}: sizes {self.nats} fail the peer-memory variant's "
                                           f"preconditions {st['pre']} (no fallback reads peers)")
                chosen = st["fallback"]
            fmad = fmad or bool(chosen.get("fmad", False))
            name_expr = f"{chosen['name']}<{targs}>" if targs else chosen["name"]
            exprs.append(name_expr)
            # a template reads / writes its buffers with 16-byte accesses (float4,
            # bulk copies, TMA): its generic kernel is compiled beside it and runs
            # instead when a caller's buffer is not 16-byte aligned (e.g. x[1:])
            # (compiled on first use: some generic kernels only compile at small sizes)
            fb = chosen.get("fallback") if chosen is st and not (
                st.get("peer_ranks") or st.get("peer_halo") or st.get("peer_out")) else None
            self.launches.append((chosen, name_expr, fb))
        self._opts = ["--fmad=true" if fmad else "--fmad=false"]
        self.module = rt.load_module(text, exprs, self._opts, program_name=f"{self.plan['unit']}.cu")
        self.kernels = []
        for (chosen, _e, _fb), lowered in zip(self.launches, self.module.lowered):
            fn = self.module.function(lowered)
            grid, block, smem, cluster = self._config(chosen)
            self.kernels.append((chosen, fn, grid, block, smem, cluster))
        self._fallbacks = {}
        self._targs = targs
        self._temps = None
        # an executable with temporaries or workspaces (launch counters, partial
        # slots, K-split flags) carries state from one launch to the next:
        # launch() keeps its launches in order across streams (SURVEY §8 b:
        # thread-safe per stream) — a launch on a stream other than the last
        # one's waits for the last one (device-side, no host sync)
        self._stateful = bool(self.plan["temps"]) or any(st.get("workspace") for st, *_ in self.kernels)
        self._order_lock = threading.Lock()
        self._temps_lock = threading.Lock()
        self._order_event = None
        self._last_stream = None

    def _fallback(self, k):
        """Stage k's generic kernel (None for a stage without one)."""
        if k not in self._fallbacks:
            with self._temps_lock:  # (compiled once even when threads race here)
                if k not in self._fallbacks:
                    fb = self.launches[k][2]
                    entry = None
                    if fb is not None:
                        expr = f"{fb['name']}<{self._targs}>" if self._targs else fb["name"]
                        mod = rt.load_module(self.text, [expr], self._opts, program_name=f"{self.plan['unit']}.cu")
                        entry = (fb, mod.function(mod.lowered[0]), *self._config(fb))
                        self._fallback_modules = getattr(self, "_fallback_modules", []) + [mod]
                    self._fallbacks[k] = entry
        return self._fallbacks[k]

    # launch configuration --------------------------------------------------
    def _config(self, st):
        kind = st["kind"]
        sm = self.sm_count
        if kind == "grid":
            total = eval_py(st["total"], self.nats)
            block = st["block"]
            grid = max(1, min(math.ceil(total / block), sm * 8))
            return (grid, 1, 1), (block, 1, 1), 0, (1, 1, 1)
        if kind == "workgroup":
            total = eval_py(st["total"], self.nats)
            locals_ = [eval_py(b, self.nats) for b in st.get("local_bounds", [])]
            want = max(locals_) if locals_ else st["block"]
            block = min(st["block"], max(32, 32 * math.ceil(want / 32)))
            grid = max(1, min(total, sm * 16))
            return (grid, 1, 1), (block, 1, 1), 0, (1, 1, 1)
        if kind == "block":
            return (1, 1, 1), (st["block"], 1, 1), 0, (1, 1, 1)
        if kind == "serial":
            return (1, 1, 1), (1, 1, 1), 0, (1, 1, 1)
        launcher = _launchers().get(kind)
        if launcher is None:
            raise InterpreterError(f"no launcher for stage kind {kind!r}")
        return launcher(st, self.nats, sm)

    @property
    def kernel_names(self):
        return [st["name"] for st, *_ in self.kernels]

    @property
    def template_kinds(self):
        return [st["kind"] for st, *_ in self.kernels]

    def temps(self):
        """Device temporaries (allocated once per executable; thread-safe: the
        table is published only once complete and its zero-fill finished)."""
        if self._temps is None:
            with self._temps_lock:
                if self._temps is None:
                    self._temps = self._alloc_temps()
        return self._temps

    def _alloc_temps(self):
        import torch

        # temporaries with disjoint stage lifetimes share a slot (plan "slot",
        # emit_cuda.reuse_slots): one allocation of the largest, viewed per type
        sizes = {}
        for t in self.plan["temps"]:
            k = t.get("slot", t["name"])
            sizes[k] = max(sizes.get(k, 1), self.temp_sizes[t["name"]])
        slots = {k: torch.empty(n, dtype=torch.float32, device="cuda") for k, n in sizes.items()}
        temps = {}
        for t in self.plan["temps"]:
            buf = slots[t.get("slot", t["name"])][: max(1, self.temp_sizes[t["name"]])]
            temps[t["name"]] = buf if t["ctype"] == "float" else buf.view(_torch_dtype(t["ctype"]))
        for st, *_ in self.kernels:
            for ws in st.get("workspace", []):
                size = eval_py(ws["size"], self.nats)
                temps[ws["name"]] = torch.zeros(max(1, size), dtype=_torch_dtype(ws["ctype"]), device="cuda")
        # the workspaces' zero-fill ran on this thread's current stream; launches may
        # come from any stream
        torch.cuda.current_stream().synchronize()
        return temps

    def _stages_for(self, buffers: dict):
        """The kernels to launch for these buffers: each template stage, or its
        generic fallback when a caller buffer is not 16-byte aligned."""
        names = [i["name"] for i in self.plan["inputs"] if not i["scalar"] and not i.get("peer")]
        names.append(self.plan["output"]["name"])
        aligned = all(_dptr(buffers[nm]) % 16 == 0 for nm in names if nm in buffers)
        if aligned:
            return self.kernels
        out = []
        for k, kern in enumerate(self.kernels):
            fb = self._fallback(k) if kern[0].get("fallback") is not None else None
            out.append(fb if fb is not None else kern)
        return out

    def launch(self, buffers: dict, stream=None):
        """Launch every stage.  `buffers` maps argument names to device
        tensors / pointers (arrays) or Python numbers (scalar inputs)."""
        temps = self.temps()
        scalar_types = {i["name"]: i["ctype"] for i in self.plan["inputs"] if i["scalar"]}
        base_args = []
        for name in self.plan["args"]:
            if name in temps:
                base_args.append(ctypes.c_void_p(temps[name].data_ptr()))
            elif name in scalar_types:
                v = buffers[name]
                base_args.append(ctypes.c_float(float(v)) if scalar_types[name] == "float" else ctypes.c_int(int(v)))
            else:
                base_args.append(ctypes.c_void_p(_dptr(buffers[name])))
        stages = []
        for st, fn, grid, block, smem, cluster in self._stages_for(buffers):
            args = list(base_args)
            for extra in st.get("extra_args", []):
                args.append(self._extra_arg(extra, buffers, temps))
            stages.append((st, fn, grid, block, smem, cluster, args))
        if not self._stateful:
            for st, fn, grid, block, smem, cluster, args in stages:
                fn.launch(grid, block, args, smem=smem, stream=stream, cluster=cluster, flags=_launch_flags(st))
            return
        key = rt.stream_key(stream)
        with self._order_lock:
            if self._order_event is None:
                self._order_event = rt.Event()
            elif key != self._last_stream:
                self._order_event.wait_on(stream)  # the previous launch on another stream first
            for st, fn, grid, block, smem, cluster, args in stages:
                fn.launch(grid, block, args, smem=smem, stream=stream, cluster=cluster, flags=_launch_flags(st))
            self._order_event.record(stream)
            self._last_stream = key

    def bind(self, buffers: dict, stream=None):
        """Pre-build every launch (argument arrays, tensor maps) for fixed
        buffers; the returned callable just issues rs_launch per stage —
        the low-overhead path for repeated steps (benchmarks, CUDA graphs)."""
        temps = self.temps()
        scalar_types = {i["name"]: i["ctype"] for i in self.plan["inputs"] if i["scalar"]}
        base_args = []
        for name in self.plan["args"]:
            if name in temps:
                base_args.append(ctypes.c_void_p(temps[name].data_ptr()))
            elif name in scalar_types:
                v = buffers[name]
                base_args.append(ctypes.c_float(float(v)) if scalar_types[name] == "float" else ctypes.c_int(int(v)))
            else:
                base_args.append(ctypes.c_void_p(_dptr(buffers[name])))
        prepared = []
        for st, fn, grid, block, smem, cluster in self._stages_for(buffers):
            args = list(base_args) + [self._extra_arg(e, buffers, temps) for e in st.get("extra_args", [])]
            prepared.append(rt.PreparedLaunch(fn, grid, block, args, smem, stream, cluster, _launch_flags(st)))

        def launch_all():
            for p in prepared:
                p()

        launch_all.prepared = prepared
        return launch_all

    def graph(self, buffers: dict, stream):
        """bind() captured into a CUDA graph: one launch replays every stage
        of the unit (`stream` must be a non-default stream)."""
        launch_all = self.bind(buffers, stream)
        g = rt.Graph(launch_all, stream)
        g.prepared = launch_all.prepared  # keep the argument arrays alive
        return g

    def _extra_arg(self, extra, buffers, temps):
        kind = extra["kind"]
        if kind == "workspace":
            return ctypes.c_void_p(temps[extra["name"]].data_ptr())
        if kind == "tma2d":
            base = _dptr(buffers[extra["buf"]]) if extra["buf"] in buffers else temps[extra["buf"]].data_ptr()
            base += 4 * eval_py(extra.get("offset", "0"), self.nats)
            dims = [eval_py(d, self.nats) for d in extra["dims"]]
            pitch = eval_py(extra.get("pitch", extra["dims"][0]), self.nats)
            box = [eval_py(str(b), self.nats) for b in extra["box"]]
            return rt.tma_desc_2d_f32(base, dims[0], dims[1], pitch * 4, box[0], box[1],
                                      extra.get("swizzle", 0))
        if kind == "peer_ptr":  # optional: absent / None / 0 -> NULL (e.g. the image's real edge)
            value = buffers.get(extra["name"])
            return ctypes.c_void_p(0 if value is None else _dptr(value) if hasattr(value, "data_ptr") else int(value))
        if kind == "peer_ptr_table":  # e.g. rs_y_table: R peer pointers + this rank's offset (int64 tensor)
            table = buffers.get(extra["name"])
            if table is None:
                raise InterpreterError(f"peer-output kernel launched without buffers[{extra['name']!r}]")
            return ctypes.c_void_p(_dptr(table))
        if kind == "peer_table":
            table = buffers.get("rs_peer_table")
            if table is None:
                raise InterpreterError("peer-source kernel launched without buffers['rs_peer_table']")
            return ctypes.c_void_p(_dptr(table))
        if kind in ("gemm_units", "gemm_full_tiles", "gemm_ksplit"):
            from .tmpl_gemm import schedule, work_units

            M, N, K = (eval_py(extra[k], self.nats) for k in ("M", "N", "K"))
            if kind == "gemm_units":
                return ctypes.c_int(work_units(M, N, K, extra["bn"], self.sm_count))
            nfull, s = schedule(M, N, K, extra["bn"], self.sm_count)
            return ctypes.c_int(nfull if kind == "gemm_full_tiles" else s)
        raise InterpreterError(f"unknown extra kernel argument {kind!r}")

    def run_host(self, host_inputs, host_out, device_inputs, device_out, stream=None, extra=None):
        """End-to-end step through host memory: copy `host_inputs` (pinned
        torch CPU tensors, scalars passed through) into `device_inputs`,
        launch, and copy the result back into `host_out` — all enqueued on
        `stream`.  The caller synchronises."""
        import torch

        stream = stream if stream is not None else torch.cuda.current_stream()
        with torch.cuda.stream(stream):
            for h, d in zip(host_inputs, device_inputs):
                if isinstance(d, torch.Tensor):
                    d.copy_(h, non_blocking=True)
            self(*device_inputs, out=device_out, stream=stream, extra=extra)
            host_out.copy_(device_out, non_blocking=True)
        return host_out

    def stream_host(self, host_steps, host_outs, depth=2, timed=False, extra=None):
        """End-to-end processing of a stream of steps from host memory:
        step k copies host_steps[k] (pinned CPU tensors / scalars, unit input
        order) to the device, runs the kernels, and copies the result into
        host_outs[k] (pinned).  The three phases run on three streams over
        `depth` device buffer sets, so step k+1's host->device copy and step
        k-1's device->host copy overlap step k's kernels (PCIe is full
        duplex): the steady state costs max(H2D, kernels, D2H) per step
        instead of their sum.  Every step still moves all of its inputs and
        its whole result through host memory.  Returns after the last copy
        has landed; with timed=True also the device time (ms, CUDA events)
        from the first copy's start to the last copy's end."""
        import torch

        specs = self.plan["inputs"]
        dev = [[torch.empty(self.input_sizes[sp["name"]], dtype=_torch_dtype(sp["ctype"]), device="cuda")
                if not sp["scalar"] else None for sp in specs] for _ in range(depth)]
        outs = [torch.empty(self.output_size, dtype=_torch_dtype(self.plan["output"]["ctype"]), device="cuda")
                for _ in range(depth)]
        launches = []
        for slot in range(depth):
            buffers = dict(extra or {})
            buffers[self.plan["output"]["name"]] = outs[slot]
            for sp, d in zip(specs, dev[slot]):
                if d is not None:
                    buffers[sp["name"]] = d
            launches.append(buffers)
        s_in, s_run, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
        ev = lambda: torch.cuda.Event()  # noqa: E731
        copied, ran, landed = [ev() for _ in range(depth)], [ev() for _ in range(depth)], [ev() for _ in range(depth)]
        used = [False] * depth
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0.record(s_in)
        for k, (hin, hout) in enumerate(zip(host_steps, host_outs)):
            slot = k % depth
            with torch.cuda.stream(s_in):
                if used[slot]:
                    s_in.wait_event(ran[slot])  # the kernels of step k - depth read these inputs
                for sp, h, d in zip(specs, hin, dev[slot]):
                    if d is not None:
                        d.copy_(h, non_blocking=True)
                copied[slot].record(s_in)
            with torch.cuda.stream(s_run):
                s_run.wait_event(copied[slot])
                if used[slot]:
                    s_run.wait_event(landed[slot])  # step k - depth's result has left this buffer
                buffers = dict(launches[slot])
                for sp, h in zip(specs, hin):
                    if sp["scalar"]:
                        buffers[sp["name"]] = h
                self.launch(buffers, stream=s_run)
                ran[slot].record(s_run)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ran[slot])
                hout.copy_(outs[slot], non_blocking=True)
                landed[slot].record(s_out)
            used[slot] = True
        t1.record(s_out)
        s_out.synchronize()
        if timed:
            return host_outs, t0.elapsed_time(t1)
        return host_outs

    # convenience: torch in / torch out -----------------------------------------
    def __call__(self, *inputs, out=None, stream=None, extra=None):
        """`extra`: additional named launch buffers (e.g. `rs_peer_table`, the
        device table of peer source pointers of a peer_ranks emission)."""
        import torch

        if len(inputs) != len(self.plan["inputs"]):
            raise InterpreterError(f"expected {len(self.plan['inputs'])} inputs, got {len(inputs)}")
        buffers = dict(extra or {})
        for spec, value in zip(self.plan["inputs"], inputs):
            if spec["scalar"]:
                buffers[spec["name"]] = value
                continue
            if not (isinstance(value, torch.Tensor) and value.is_cuda):
                raise InterpreterError(f"input {spec['name']!r} must be a CUDA tensor")
            if spec.get("peer"):  # read through rs_peer_table; the local argument is this rank's block
                buffers[spec["name"]] = value
                continue
            if value.numel() != self.input_sizes[spec["name"]]:
                raise InterpreterError(
                    f"input {spec['name']!r} has {value.numel()} elements, expected {self.input_sizes[spec['name']]}")
            if not value.is_contiguous() or value.dtype != _torch_dtype(spec["ctype"]):
                raise InterpreterError(f"input {spec['name']!r} must be contiguous {spec['ctype']}")
            buffers[spec["name"]] = value
        if out is None:
            out = torch.empty(self.output_size, dtype=_torch_dtype(self.plan["output"]["ctype"]), device="cuda")
        buffers[self.plan["output"]["name"]] = out
        self.launch(buffers, stream=stream if stream is not None else torch.cuda.current_stream())
        return out


def _launch_flags(st) -> int:
    return (1 if st.get("cooperative") else 0) | (2 if st.get("pdl") else 0)  # RS_LAUNCH_COOPERATIVE | _PDL


def _dptr(x):
    if hasattr(x, "data_ptr"):
        return int(x.data_ptr())
    if isinstance(x, ctypes.c_void_p):
        return int(x.value)
    if isinstance(x, rt.DeviceBuffer):
        return int(x.ptr.value)
    return int(x)


def _torch_dtype(ctype):
    import torch

    return torch.float32 if ctype == "float" else torch.int32


def _np_dtype(ctype):
    return np.float32 if ctype == "float" else np.int32


_exe_cache: dict = {}


def executable(code, nats: dict) -> Executable:
    text = code.text if isinstance(code, CudaCode) else code
    key = (text, tuple(sorted((k, int(v)) for k, v in nats.items())))
    exe = _exe_cache.get(key)
    if exe is None:
        exe = Executable(text, nats)
        _exe_cache[key] = exe
    return exe


def flatten_input(raw, dtype, nat_env):
    """Reference value (nested lists) or numpy array -> flat numpy array."""
    if isinstance(dtype, ScalarType):
        return interpreter.convert_input(raw, dtype)
    dims = []
    dt = dtype
    while isinstance(dt, ArrayType):
        dims.append(nat.evaluate(dt.size, nat_env))
        dt = dt.elem
    if not isinstance(dt, ScalarType):
        raise InterpreterError("tuple-typed kernel data has no flat layout")
    np_t = np.float32 if dt.name == "f32" else np.int32
    if isinstance(raw, np.ndarray):
        arr = np.ascontiguousarray(raw, dtype=np_t)
        if arr.size != int(np.prod(dims)):
            raise InterpreterError(f"input of {arr.size} elements does not match {dims}")
        return arr.reshape(-1)
    value = interpreter.convert_input(raw, dtype)
    interpreter.check_length(value, dtype, nat_env)
    return np.asarray(value, dtype=np_t).reshape(-1)


def unflatten(flat: np.ndarray, dtype, nat_env):
    dims = []
    dt = dtype
    while isinstance(dt, ArrayType):
        dims.append(nat.evaluate(dt.size, nat_env))
        dt = dt.elem
    if not dims:
        v = flat[0]
        return np.float32(v) if flat.dtype == np.float32 else int(v)
    arr = flat.reshape(dims)
    if flat.dtype == np.float32:
        return _to_nested(arr, np.float32)
    return _to_nested(arr, int)


def _to_nested(arr, conv):
    if arr.ndim == 1:
        return [conv(v) for v in arr]
    return [_to_nested(a, conv) for a in arr]


def run_cuda(code, unit, nat_assignment: dict, inputs, *, stream=None, as_numpy=False, as_device=False):
    """Execute sm100a kernel text for a translated unit on the GPU and return
    its output in the interpreter's nested-value form (or a flat numpy array
    with `as_numpy=True`, or the flat device tensor itself with
    `as_device=True`: no copy back, the caller synchronises).  Same contract
    as cexec.run_emitted (cexec.py:555): inputs in unit order, sizes by
    name, output allocated here.  Inputs may be the reference's nested
    values, numpy arrays, or torch tensors (a contiguous CUDA tensor of the
    right dtype and size is used in place: the zero-copy path)."""
    import torch

    nat_env = {k: int(v) for k, v in dict(nat_assignment).items()}
    exe = executable(code, nat_env)
    if len(inputs) != len(unit.inputs):
        raise InterpreterError(f"expected {len(unit.inputs)} inputs, got {len(inputs)}")
    dev_inputs = []
    for (var, dtype), raw in zip(unit.inputs, inputs):
        if isinstance(raw, torch.Tensor) and not isinstance(dtype, ScalarType):
            if raw.is_cuda:
                dev_inputs.append(raw.reshape(-1))  # Executable checks size, dtype, contiguity
                continue
            raw = raw.numpy()
        flat = flatten_input(raw, dtype, nat_env)
        if isinstance(dtype, ScalarType):
            dev_inputs.append(flat)
        else:
            dev_inputs.append(torch.from_numpy(np.ascontiguousarray(flat)).to("cuda"))
    out = exe(*dev_inputs, stream=stream)
    if as_device:
        return out
    torch.cuda.synchronize()
    host = out.cpu().numpy()
    if as_numpy:
        return host
    return unflatten(host, unit.output_type, nat_env)
