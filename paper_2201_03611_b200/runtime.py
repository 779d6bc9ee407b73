"""ctypes binding of the native runtime (include/rise_b200.h).

This is the Python half of the drop-in boundary.  Compile failures raise the
reference's `EmitError` (stage "emit", errors.py:73-74); launch, memory and
device failures raise `InterpreterError` (stage "run", errors.py:77-78), the
classes `codegen.emit` and `cexec.execute_kernel` raise today.

There is no fallback: if the shared library or the CUDA driver is missing,
every entry point that needs them raises.
"""

from __future__ import annotations

import ctypes
import hashlib
import os
import threading
from pathlib import Path

from ._ref import errors as _errors

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "_lib" / "librise_b200.so"
INCLUDE_DIR = PKG_DIR / "csrc" / "include"
HEADER = PKG_DIR.parent / "include" / "rise_b200.h"

# every symbol include/rise_b200.h declares (checked by the CPU test-suite)
EXPORTED = (
    "rs_last_error", "rs_abi_version", "rs_init", "rs_device_count", "rs_device_attribute",
    "rs_nvrtc_version", "rs_compile", "rs_compile_cubin", "rs_free_host", "rs_module_load",
    "rs_module_lowered_name", "rs_module_get_function", "rs_module_unload",
    "rs_function_attribute", "rs_launch", "rs_launch_ex", "rs_malloc", "rs_free", "rs_memcpy_htod",
    "rs_memcpy_dtoh", "rs_memcpy_dtod", "rs_memcpy_peer", "rs_memset_d8", "rs_stream_create",
    "rs_stream_destroy", "rs_stream_synchronize", "rs_device_synchronize", "rs_event_create",
    "rs_event_destroy", "rs_event_record", "rs_event_synchronize", "rs_event_elapsed_ms",
    "rs_stream_wait_event", "rs_tma_desc_2d_f32", "rs_ipc_handle", "rs_ipc_open", "rs_ipc_close", "rs_halo_exchange",
    "rs_comm_unique_id", "rs_comm_init", "rs_comm_destroy", "rs_allgather",
    "rs_graph_capture_begin", "rs_graph_capture_end", "rs_graph_launch", "rs_graph_upload", "rs_graph_destroy",
)

_lib = None
_lock = threading.Lock()


class RuntimeUnavailable(_errors.InterpreterError):
    """The native runtime library could not be loaded."""


def lib():
    """Load librise_b200.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise RuntimeUnavailable(
                    f"native runtime {LIB_PATH} is missing; run __graft_entry__.build()"
                )
            L = ctypes.CDLL(str(LIB_PATH))
            vp, i, sz, u = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t, ctypes.c_uint
            cpp = ctypes.POINTER(ctypes.c_char_p)
            L.rs_last_error.restype = ctypes.c_char_p
            L.rs_abi_version.restype = i
            L.rs_compile_cubin.argtypes = [ctypes.c_char_p, ctypes.c_char_p, cpp, i, cpp, i,
                                           ctypes.POINTER(vp), ctypes.POINTER(sz),
                                           ctypes.POINTER(vp), ctypes.POINTER(vp)]
            L.rs_free_host.argtypes = [vp]
            L.rs_free_host.restype = None
            L.rs_module_load.argtypes = [vp, sz, ctypes.POINTER(vp)]
            L.rs_module_get_function.argtypes = [vp, ctypes.c_char_p, ctypes.POINTER(vp)]
            L.rs_module_unload.argtypes = [vp]
            L.rs_function_attribute.argtypes = [vp, i, ctypes.POINTER(i)]
            L.rs_launch.argtypes = [vp, ctypes.POINTER(u), ctypes.POINTER(u), ctypes.POINTER(u),
                                    u, vp, ctypes.POINTER(vp)]
            L.rs_launch_ex.argtypes = [vp, ctypes.POINTER(u), ctypes.POINTER(u), ctypes.POINTER(u),
                                       u, vp, ctypes.POINTER(vp), u]
            L.rs_malloc.argtypes = [ctypes.POINTER(vp), sz]
            L.rs_free.argtypes = [vp]
            for name in ("rs_memcpy_htod", "rs_memcpy_dtoh", "rs_memcpy_dtod"):
                getattr(L, name).argtypes = [vp, vp, sz, vp]
            L.rs_memset_d8.argtypes = [vp, ctypes.c_ubyte, sz, vp]
            L.rs_memcpy_peer.argtypes = [vp, i, vp, i, sz, vp]
            L.rs_stream_create.argtypes = [ctypes.POINTER(vp)]
            L.rs_stream_destroy.argtypes = [vp]
            L.rs_stream_synchronize.argtypes = [vp]
            L.rs_event_create.argtypes = [ctypes.POINTER(vp)]
            L.rs_event_destroy.argtypes = [vp]
            L.rs_event_record.argtypes = [vp, vp]
            L.rs_event_synchronize.argtypes = [vp]
            L.rs_event_elapsed_ms.argtypes = [ctypes.POINTER(ctypes.c_float), vp, vp]
            L.rs_stream_wait_event.argtypes = [vp, vp]
            L.rs_tma_desc_2d_f32.argtypes = [vp, vp, ctypes.c_uint64, ctypes.c_uint64,
                                             ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, i]
            L.rs_device_attribute.argtypes = [i, ctypes.POINTER(i)]
            L.rs_device_count.argtypes = [ctypes.POINTER(i)]
            L.rs_nvrtc_version.argtypes = [ctypes.POINTER(i), ctypes.POINTER(i)]
            L.rs_ipc_handle.argtypes = [vp, ctypes.POINTER(sz), vp]
            L.rs_ipc_open.argtypes = [ctypes.POINTER(vp), vp, sz]
            L.rs_ipc_close.argtypes = [vp]
            L.rs_halo_exchange.argtypes = [vp, sz, sz, vp, sz, vp, vp]
            L.rs_comm_unique_id.argtypes = [vp]
            L.rs_comm_init.argtypes = [ctypes.POINTER(vp), i, i, vp]
            L.rs_comm_destroy.argtypes = [vp]
            L.rs_allgather.argtypes = [vp, vp, vp, sz, vp]
            L.rs_graph_capture_begin.argtypes = [vp]
            L.rs_graph_capture_end.argtypes = [vp, ctypes.POINTER(vp)]
            L.rs_graph_launch.argtypes = [vp, vp]
            L.rs_graph_upload.argtypes = [vp, vp]
            L.rs_graph_destroy.argtypes = [vp]
            _lib = L
    return _lib


def _err_text():
    return lib().rs_last_error().decode(errors="replace")


def check_run(status, what=""):
    if status != 0:
        raise _errors.InterpreterError(f"{what}: {_err_text()}" if what else _err_text())


def _cstr_array(items):
    arr = (ctypes.c_char_p * max(1, len(items)))()
    for k, s in enumerate(items):
        arr[k] = s.encode()
    return arr


# ---------------------------------------------------------------------------
# compilation (device-independent)

DEFAULT_OPTS = ("--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo", "-default-device")

_cubin_cache: dict = {}
_headers_digest = None


def _include_digest() -> str:
    """Hash of the device headers the kernel text includes (part of the
    cache key: a changed header is a different cubin)."""
    global _headers_digest
    if _headers_digest is None:
        h = hashlib.sha256()
        for p in sorted(Path(INCLUDE_DIR).rglob("*")):
            if p.is_file():
                h.update(p.name.encode())
                h.update(p.read_bytes())
        _headers_digest = h.hexdigest()
    return _headers_digest


def cache_dir():
    """On-disk cubin cache keyed by the source hash (RISE_CUBIN_CACHE; "0"
    disables it).  Only a compile-time saving: a miss recompiles."""
    d = os.environ.get("RISE_CUBIN_CACHE", str(Path.home() / ".cache" / "rise_b200" / "cubin"))
    return None if d == "0" else Path(d)


def _disk_get(key):
    d = cache_dir()
    if d is None:
        return None
    try:
        blob = (d / f"{key}.cubin").read_bytes()
        names = (d / f"{key}.names").read_text().split("\n")
    except OSError:
        return None
    return blob, names


def _disk_put(key, blob, names):
    d = cache_dir()
    if d is None:
        return
    try:
        d.mkdir(parents=True, exist_ok=True)
        for suffix, data in ((".names", "\n".join(names).encode()), (".cubin", blob)):
            tmp = d / f"{key}{suffix}.{os.getpid()}.tmp"
            tmp.write_bytes(data)
            os.replace(tmp, d / f"{key}{suffix}")  # atomic: concurrent ranks may race
    except OSError:
        pass


def compile_cubin(source: str, name_exprs, opts=(), program_name="rise.cu"):
    """NVRTC-compile `source` for sm_100a.  Returns (cubin bytes, lowered names).
    Raises EmitError with the NVRTC log on failure.  Needs no GPU."""
    full_opts = list(DEFAULT_OPTS) + [f"-I{INCLUDE_DIR}"] + list(opts)
    key = hashlib.sha256(
        "\0".join([source, program_name, _include_digest()] + full_opts + list(name_exprs)).encode()
    ).hexdigest()
    hit = _cubin_cache.get(key)
    if hit is not None:
        return hit
    hit = _disk_get(key)
    if hit is not None and len(hit[1]) == len(name_exprs):
        _cubin_cache[key] = hit
        return hit
    L = lib()
    image, size = ctypes.c_void_p(), ctypes.c_size_t()
    names, log = ctypes.c_void_p(), ctypes.c_void_p()
    st = L.rs_compile_cubin(
        source.encode(), program_name.encode(), _cstr_array(full_opts), len(full_opts),
        _cstr_array(list(name_exprs)), len(name_exprs),
        ctypes.byref(image), ctypes.byref(size), ctypes.byref(names), ctypes.byref(log),
    )
    if st != 0:
        raise _errors.EmitError(_err_text())
    try:
        blob = ctypes.string_at(image, size.value)
        lowered = ctypes.string_at(names).decode().split("\n")[: len(name_exprs)] if names else []
    finally:
        L.rs_free_host(image)
        L.rs_free_host(names)
        L.rs_free_host(log)
    out = (blob, lowered)
    _cubin_cache[key] = out
    _disk_put(key, blob, lowered)
    return out


# ---------------------------------------------------------------------------
# device side

_device = None


def init(device: int | None = None):
    """Make `device`'s primary context current (default: torch's current
    device if torch has initialised CUDA, else 0)."""
    global _device
    if device is None:
        device = _device if _device is not None else int(os.environ.get("LOCAL_RANK", "0") or 0)
        try:
            import torch

            if torch.cuda.is_available() and torch.cuda.is_initialized():
                device = torch.cuda.current_device()
        except Exception:  # noqa: BLE001 - torch is optional plumbing
            pass
    check_run(lib().rs_init(int(device)), "rs_init")
    _device = int(device)
    return _device


def device_attribute(attr: int) -> int:
    init()
    v = ctypes.c_int()
    check_run(lib().rs_device_attribute(attr, ctypes.byref(v)), "rs_device_attribute")
    return v.value


SM_COUNT_ATTR = 16


class Module:
    def __init__(self, cubin: bytes, lowered):
        init()
        self._handle = ctypes.c_void_p()
        self._image = ctypes.create_string_buffer(cubin, len(cubin))
        check_run(lib().rs_module_load(self._image, len(cubin), ctypes.byref(self._handle)),
                  "rs_module_load")
        self.lowered = list(lowered)
        self._fns = {}

    def function(self, lowered_name: str) -> "Function":
        fn = self._fns.get(lowered_name)
        if fn is None:
            h = ctypes.c_void_p()
            check_run(lib().rs_module_get_function(self._handle, lowered_name.encode(), ctypes.byref(h)),
                      "rs_module_get_function")
            fn = Function(h, lowered_name)
            self._fns[lowered_name] = fn
        return fn


class Function:
    def __init__(self, handle, name):
        self.handle = handle
        self.name = name

    def attribute(self, attr: int) -> int:
        v = ctypes.c_int()
        check_run(lib().rs_function_attribute(self.handle, attr, ctypes.byref(v)), "rs_function_attribute")
        return v.value

    def launch(self, grid, block, args, smem=0, stream=None, cluster=(1, 1, 1), flags=0):
        """`args`: list of ctypes values (kept alive for the call); `flags`:
        RS_LAUNCH_COOPERATIVE (1) / RS_LAUNCH_PDL (2) of rs_launch_ex."""
        g = (ctypes.c_uint * 3)(*_dim3(grid))
        b = (ctypes.c_uint * 3)(*_dim3(block))
        c = (ctypes.c_uint * 3)(*_dim3(cluster))
        ptrs = (ctypes.c_void_p * max(1, len(args)))()
        for k, a in enumerate(args):
            ptrs[k] = ctypes.cast(ctypes.byref(a), ctypes.c_void_p)
        check_run(
            lib().rs_launch_ex(self.handle, g, b, c, int(smem), _stream_ptr(stream), ptrs, int(flags)),
            f"launch of {self.name}",
        )


class PreparedLaunch:
    """One kernel launch with its argument array built once."""

    def __init__(self, fn: Function, grid, block, args, smem=0, stream=None, cluster=(1, 1, 1), flags=0):
        self.fn = fn
        self.flags = int(flags)
        self.args = list(args)  # keep the ctypes values alive
        self.g = (ctypes.c_uint * 3)(*_dim3(grid))
        self.b = (ctypes.c_uint * 3)(*_dim3(block))
        self.c = (ctypes.c_uint * 3)(*_dim3(cluster))
        self.ptrs = (ctypes.c_void_p * max(1, len(self.args)))()
        for k, a in enumerate(self.args):
            self.ptrs[k] = ctypes.cast(ctypes.byref(a), ctypes.c_void_p)
        self.smem = int(smem)
        self.stream = _stream_ptr(stream)
        self._launch = lib().rs_launch_ex

    def __call__(self):
        if self._launch(self.fn.handle, self.g, self.b, self.c, self.smem, self.stream, self.ptrs, self.flags) != 0:
            check_run(1, f"launch of {self.fn.name}")


def _dim3(d):
    if isinstance(d, int):
        return (d, 1, 1)
    d = tuple(int(x) for x in d)
    return d + (1,) * (3 - len(d))


def stream_key(stream):
    """A hashable identity of a stream argument (None: the legacy default stream)."""
    p = _stream_ptr(stream)
    return None if p is None else (p.value if isinstance(p, ctypes.c_void_p) else int(p))


def _stream_ptr(stream):
    if stream is None:
        return None
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    h = getattr(stream, "cuda_stream", None)
    if h is not None:
        return ctypes.c_void_p(int(h))
    return stream


_modules: dict = {}


def load_module(source: str, name_exprs, opts=(), program_name="rise.cu") -> Module:
    key = (source, tuple(name_exprs), tuple(opts))
    mod = _modules.get(key)
    if mod is None:
        cubin, lowered = compile_cubin(source, name_exprs, opts, program_name)
        mod = Module(cubin, lowered)
        _modules[key] = mod
    return mod


# memory helpers ------------------------------------------------------------


class DeviceBuffer:
    """A raw device allocation owned by the runtime (rs_malloc/rs_free)."""

    def __init__(self, nbytes: int):
        init()
        self.nbytes = int(nbytes)
        self.ptr = ctypes.c_void_p()
        check_run(lib().rs_malloc(ctypes.byref(self.ptr), self.nbytes), "rs_malloc")

    def __del__(self):
        try:
            if self.ptr and _lib is not None:
                _lib.rs_free(self.ptr)
        except Exception:  # noqa: BLE001
            pass


def memcpy_htod(dst, src_host_ptr, nbytes, stream=None):
    check_run(lib().rs_memcpy_htod(_vp(dst), _vp(src_host_ptr), nbytes, _stream_ptr(stream)), "htod")


def memcpy_dtoh(dst_host_ptr, src, nbytes, stream=None):
    check_run(lib().rs_memcpy_dtoh(_vp(dst_host_ptr), _vp(src), nbytes, _stream_ptr(stream)), "dtoh")


def memcpy_peer(dst, dst_device, src, src_device, nbytes, stream=None):
    """Device-to-device copy between two GPUs of the node (NVLink / NVSwitch)."""
    check_run(lib().rs_memcpy_peer(_vp(dst), int(dst_device), _vp(src), int(src_device), nbytes,
                                   _stream_ptr(stream)), "rs_memcpy_peer")


def memset_d8(dst, value, nbytes, stream=None):
    check_run(lib().rs_memset_d8(_vp(dst), value, nbytes, _stream_ptr(stream)), "memset")


def stream_synchronize(stream=None):
    check_run(lib().rs_stream_synchronize(_stream_ptr(stream)), "stream sync")


def _vp(p):
    if isinstance(p, ctypes.c_void_p):
        return p
    if isinstance(p, DeviceBuffer):
        return p.ptr
    return ctypes.c_void_p(int(p))


class Event:
    def __init__(self):
        init()
        self.h = ctypes.c_void_p()
        check_run(lib().rs_event_create(ctypes.byref(self.h)), "event create")

    def record(self, stream=None):
        check_run(lib().rs_event_record(self.h, _stream_ptr(stream)), "event record")

    def synchronize(self):
        check_run(lib().rs_event_synchronize(self.h), "event sync")

    def wait_on(self, stream=None):
        """Make work enqueued on `stream` from now on wait for this event."""
        check_run(lib().rs_stream_wait_event(_stream_ptr(stream), self.h), "stream wait event")

    def elapsed_ms(self, end: "Event") -> float:
        v = ctypes.c_float()
        check_run(lib().rs_event_elapsed_ms(ctypes.byref(v), self.h, end.h), "elapsed")
        return float(v.value)


def tma_desc_2d_f32(base_ptr, dim0, dim1, row_stride_bytes, box0, box1, swizzle=0):
    """Encode a CUtensorMap (128 bytes, returned as a ctypes array that can be
    passed by value as a __grid_constant__ kernel argument)."""
    desc = TensorMap()
    check_run(
        lib().rs_tma_desc_2d_f32(ctypes.byref(desc), _vp(base_ptr), dim0, dim1, row_stride_bytes,
                                 box0, box1, swizzle),
        "rs_tma_desc_2d_f32",
    )
    return desc


class TensorMap(ctypes.Structure):
    _pack_ = 64
    _fields_ = [("words", ctypes.c_uint64 * 16)]


# multi-GPU: peer memory and NCCL (include/rise_b200.h "multi-GPU") ---------


def ipc_handle(dptr):
    """(64-byte handle, offset) exporting the allocation that holds dptr."""
    init()
    h = ctypes.create_string_buffer(64)
    off = ctypes.c_size_t()
    check_run(lib().rs_ipc_handle(h, ctypes.byref(off), _vp(dptr)), "rs_ipc_handle")
    return h.raw, int(off.value)


def ipc_open(handle: bytes, offset: int) -> int:
    init()
    out = ctypes.c_void_p()
    check_run(lib().rs_ipc_open(ctypes.byref(out), ctypes.create_string_buffer(handle, 64), offset), "rs_ipc_open")
    return int(out.value)


def ipc_close(dptr):
    check_run(lib().rs_ipc_close(_vp(dptr)), "rs_ipc_close")


def halo_exchange(band_ptr, row_bytes, rows, above=None, above_rows=0, below=None, stream=None):
    check_run(lib().rs_halo_exchange(_vp(band_ptr), row_bytes, rows, _vp(above or 0), above_rows,
                                     _vp(below or 0), _stream_ptr(stream)), "rs_halo_exchange")


def comm_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    check_run(lib().rs_comm_unique_id(buf), "rs_comm_unique_id")
    return buf.raw


class NcclComm:
    """An NCCL communicator owned by the native runtime."""

    def __init__(self, nranks: int, rank: int, unique_id: bytes):
        init()
        self.h = ctypes.c_void_p()
        self.nranks, self.rank = nranks, rank
        check_run(lib().rs_comm_init(ctypes.byref(self.h), nranks, rank, ctypes.create_string_buffer(unique_id, 128)),
                  "rs_comm_init")

    def allgather(self, send_ptr, recv_ptr, bytes_per_rank, stream=None):
        check_run(lib().rs_allgather(self.h, _vp(send_ptr), _vp(recv_ptr), bytes_per_rank, _stream_ptr(stream)),
                  "rs_allgather")

    def close(self):
        if self.h:
            check_run(lib().rs_comm_destroy(self.h), "rs_comm_destroy")
            self.h = ctypes.c_void_p()


# CUDA graphs ------------------------------------------------------------------


class Graph:
    """Everything `record()` enqueues on `stream` (a torch CUDA stream or a
    raw CUstream), captured once into an executable graph; `__call__`
    replays it with a single launch on that stream."""

    def __init__(self, record, stream):
        init()
        self.stream = _stream_ptr(stream)
        self.h = ctypes.c_void_p()
        check_run(lib().rs_graph_capture_begin(self.stream), "rs_graph_capture_begin")
        try:
            record()
        finally:
            check_run(lib().rs_graph_capture_end(self.stream, ctypes.byref(self.h)), "rs_graph_capture_end")

    def __call__(self):
        check_run(lib().rs_graph_launch(self.h, self.stream), "rs_graph_launch")

    def upload(self):
        """Move the graph's work to the device now (cuGraphUpload), so the
        first replay starts without the upload."""
        check_run(lib().rs_graph_upload(self.h, self.stream), "rs_graph_upload")

    def __del__(self):
        try:
            if self.h and _lib is not None:
                _lib.rs_graph_destroy(self.h)
        except Exception:  # noqa: BLE001
            pass
