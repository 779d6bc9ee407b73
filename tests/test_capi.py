"""The C-ABI library (include/rise_b200.h) loads and exports every declared
symbol; NVRTC compilation works without a device (CPU only)."""

import ctypes
import re

import pytest

from paper_2201_03611_b200 import runtime


def _declared():
    text = runtime.HEADER.read_text()
    return sorted(set(re.findall(r"\b(rs_[a-z0-9_]+)\s*\(", text)))


def test_header_declarations_match_the_binding_list():
    assert _declared() == sorted(runtime.EXPORTED)


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(runtime.LIB_PATH))
    missing = [s for s in _declared() if not hasattr(lib, s)]
    assert not missing


def test_abi_version_and_nvrtc():
    L = runtime.lib()
    assert L.rs_abi_version() == 1
    major, minor = ctypes.c_int(), ctypes.c_int()
    assert L.rs_nvrtc_version(ctypes.byref(major), ctypes.byref(minor)) == 0
    assert (major.value, minor.value) >= (12, 8)


def test_compile_cubin_without_a_gpu():
    src = "template <int n> __global__ void k(float* o) { if (threadIdx.x < n) o[threadIdx.x] = 1.0f; }"
    cubin, lowered = runtime.compile_cubin(src, ["k<4>"])
    assert cubin[:4] == b"\x7fELF" and lowered[0].startswith("_Z")


def test_compile_error_raises_emit_error_with_log():
    from paper_2201_03611_b200._ref import errors

    with pytest.raises(errors.EmitError) as e:
        runtime.compile_cubin("__global__ void k() { this is not cuda }", ["k"])
    assert "NVRTC" in str(e.value)


def test_status_and_last_error_without_device():
    L = runtime.lib()
    st = L.rs_malloc(ctypes.byref(ctypes.c_void_p()), 16)  # no rs_init yet on this thread
    assert st != 0 and L.rs_last_error()
