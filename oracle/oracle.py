"""TEST INFRASTRUCTURE ONLY — the checker, never the product.

ctypes access to
  * oracle/_build/librise_oracle.so — the C restatement (rise_oracle.c), and
  * oracle/_ref/libref_kernels.so  — the reference's own emitted C
    (make_ref.py; bit-exact with the reference interpreter),
plus the parity rules of SURVEY.md §8 d as functions.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this module.
"""

from __future__ import annotations

import ctypes
import math
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_LIB = HERE / "_build" / "librise_oracle.so"
REF_LIB = HERE / "_ref" / "libref_kernels.so"

U = 2.0 ** -24  # unit roundoff of binary32

_fp = ctypes.POINTER(ctypes.c_float)
_dp = ctypes.POINTER(ctypes.c_double)
_i64 = ctypes.c_int64
_int = ctypes.c_int

_lib = None
_ref = None


def _ptr(a, t=_fp):
    return a.ctypes.data_as(t)


def lib():
    global _lib
    if _lib is None:
        if not ORACLE_LIB.exists():
            raise FileNotFoundError(f"{ORACLE_LIB} missing; run `make -C oracle`")
        L = ctypes.CDLL(str(ORACLE_LIB))
        L.oracle_dot.restype = ctypes.c_float
        L.oracle_dot.argtypes = [_i64, _fp, _fp]
        L.oracle_dot_f64.argtypes = [_i64, _fp, _fp, _dp, _dp]
        L.oracle_mv.argtypes = [_i64, _i64, _fp, _fp, _fp]
        L.oracle_conv3x3.argtypes = [_i64, _i64, _fp, _fp, _fp]
        L.oracle_sgemm_bt.argtypes = [_i64, _i64, _i64, _fp, _fp, _fp]
        L.oracle_sgemm_bt_f64.argtypes = [_i64, _i64, _i64, _fp, _fp, _dp, _dp]
        L.oracle_nbody.argtypes = [_i64, _fp, _fp, _fp, _fp, _i64, _i64]
        L.oracle_nbody_acc_f64.argtypes = [_i64, _fp, _fp, _dp, _i64, _i64]
        L.oracle_omp_threads.restype = _int
        _lib = L
    return _lib


def ref_lib():
    """The reference's emitted C (None when it has not been built)."""
    global _ref
    if _ref is None:
        if not REF_LIB.exists():
            return None
        L = ctypes.CDLL(str(REF_LIB))
        L.dotKernel.argtypes = [_fp, _int, _fp, _fp]
        L.mvKernel.argtypes = [_fp, _int, _int, _fp, _fp]
        L.mvOptKernel.argtypes = [_fp, _int, _int, _int, _fp, _fp]
        L.sgemmBtKernel.argtypes = [_fp, _int, _int, _int, _fp, _fp]
        L.convKernel.argtypes = [_fp, _int, _int, _fp, _fp]
        L.asumKernel.argtypes = [_fp, _int, _fp]
        L.dotChunkedKernel.argtypes = [_fp, _int, _fp, _fp]
        L.nbodyShardKernel.argtypes = [_fp, _int, _int, _fp, _fp, _fp, _fp]
        _ref = L
    return _ref


def threads():
    return int(lib().oracle_omp_threads())


def f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


# ---- C restatement -----------------------------------------------------------


def dot(a, b) -> np.float32:
    a, b = f32(a), f32(b)
    return np.float32(lib().oracle_dot(a.size, _ptr(a), _ptr(b)))


def dot_f64(a, b):
    a, b = f32(a), f32(b)
    v, s = ctypes.c_double(), ctypes.c_double()
    lib().oracle_dot_f64(a.size, _ptr(a), _ptr(b), ctypes.byref(v), ctypes.byref(s))
    return v.value, s.value


def mv(M, x):
    M, x = f32(M), f32(x)
    n, m = M.shape
    out = np.empty(n, np.float32)
    lib().oracle_mv(n, m, _ptr(M), _ptr(x), _ptr(out))
    return out


def conv3x3(img, w):
    img, w = f32(img), f32(w)
    n, m = img.shape
    out = np.empty((n, m), np.float32)
    lib().oracle_conv3x3(n, m, _ptr(img), _ptr(w), _ptr(out))
    return out


def sgemm_bt(A, Bt):
    A, Bt = f32(A), f32(Bt)
    n, k = A.shape
    m = Bt.shape[0]
    C = np.empty((n, m), np.float32)
    lib().oracle_sgemm_bt(n, m, k, _ptr(A), _ptr(Bt), _ptr(C))
    return C


def sgemm_bt_f64(A, Bt):
    A, Bt = f32(A), f32(Bt)
    n, k = A.shape
    m = Bt.shape[0]
    C = np.empty((n, m), np.float64)
    absC = np.empty((n, m), np.float64)
    lib().oracle_sgemm_bt_f64(n, m, k, _ptr(A), _ptr(Bt), _ptr(C, _dp), _ptr(absC, _dp))
    return C, absC


def nbody(pos, vel, mass, first=0, count=None):
    pos, vel, mass = f32(pos), f32(vel), f32(mass)
    n = mass.size
    count = n - first if count is None else count
    out = np.empty((count, 3), np.float32)
    lib().oracle_nbody(n, _ptr(pos), _ptr(vel), _ptr(mass), _ptr(out), first, count)
    return out


def nbody_acc_f64(pos, mass, first=0, count=None):
    pos, mass = f32(pos), f32(mass)
    n = mass.size
    count = n - first if count is None else count
    out = np.empty((count, 3), np.float64)
    lib().oracle_nbody_acc_f64(n, _ptr(pos), _ptr(mass), _ptr(out, _dp), first, count)
    return out


# ---- the reference's own emitted C ------------------------------------------


def ref_dot(a, b):
    L = ref_lib()
    a, b = f32(a), f32(b)
    out = np.zeros(1, np.float32)
    L.dotKernel(_ptr(out), a.size, _ptr(a), _ptr(b))
    return out[0]


def ref_mv(M, x, s=None):
    L = ref_lib()
    M, x = f32(M), f32(x)
    n, m = M.shape
    out = np.zeros(n, np.float32)
    if s is None:
        L.mvKernel(_ptr(out), n, m, _ptr(M), _ptr(x))
    else:
        L.mvOptKernel(_ptr(out), n, m, s, _ptr(M), _ptr(x))
    return out


def ref_dot_chunked(a, b):
    """The reference emitter's OpenMP C for DOT + the chunked-reduce strategy:
    4096-element chunk folds in parallel, then their left fold."""
    L = ref_lib()
    a, b = f32(a), f32(b)
    out = np.zeros(1, np.float32)
    L.dotChunkedKernel(_ptr(out), a.size, _ptr(a), _ptr(b))
    return out[0]


def ref_asum(x):
    """The reference emitter's C for programs.ASUM (sequential left fold of |x_i|)."""
    L = ref_lib()
    x = f32(x)
    out = np.zeros(1, np.float32)
    L.asumKernel(_ptr(out), x.size, _ptr(x))
    return out[0]


def ref_conv3x3(img, w):
    """The reference emitter's OpenMP C for programs.CONV (extension seams)."""
    L = ref_lib()
    img, w = f32(img), f32(w)
    n, m = img.shape
    out = np.zeros((n, m), np.float32)
    L.convKernel(_ptr(out), n, m, _ptr(img), _ptr(w))
    return out


def ref_nbody_block(pos, vel, mass, first, count):
    """The reference emitter's OpenMP C for programs.NBODY_SHARD: the step of
    target bodies first .. first+count-1 against all sources."""
    L = ref_lib()
    pos, vel, mass = f32(pos), f32(vel), f32(mass)
    n = mass.size
    tpos = np.ascontiguousarray(pos[first:first + count])
    tvel = np.ascontiguousarray(vel[first:first + count])
    out = np.zeros((count, 3), np.float32)
    L.nbodyShardKernel(_ptr(out), count, n, _ptr(tpos), _ptr(tvel), _ptr(pos), _ptr(mass))
    return out


def ref_sgemm_bt(A, Bt):
    L = ref_lib()
    A, Bt = f32(A), f32(Bt)
    n, k = A.shape
    m = Bt.shape[0]
    C = np.zeros((n, m), np.float32)
    L.sgemmBtKernel(_ptr(C), n, m, k, _ptr(A), _ptr(Bt))
    return C


# ---- parity rules (SURVEY.md §8 d) ---------------------------------------------


def reduction_bound(n_terms: int, abs_sum: float, slack: int = 2) -> float:
    """|y - y64| <= 2 (ceil(log2 n) + c) u sum|terms| for a reassociated
    fp32 sum of n products (tree depth + per-thread fold length)."""
    depth = math.ceil(math.log2(max(2, n_terms)))
    return 2.0 * (depth + slack) * U * abs_sum + 1e-30


def reassociated_dot_bound(n: int, abs_sum: float, per_thread: int) -> float:
    """Bound for the `reduce` template's order: a left fold of <= per_thread
    terms followed by a tree of depth log2(#partials): error <=
    (per_thread + tree_depth + 1) u sum|terms| (first order)."""
    depth = math.ceil(math.log2(max(2, -(-n // max(1, per_thread)))))
    return (per_thread + depth + 2) * U * abs_sum + 1e-30


def gemm_bound(k: int, absC):
    """|C - C64| <= 2 k u (|A||B|)_ij  (SURVEY.md §8 d, C4)."""
    return 2.0 * k * U * absC + 1e-30


def rng_inputs(seed: int, *shape, low=-1.0, high=1.0):
    return np.random.default_rng(seed).uniform(low, high, shape).astype(np.float32)


def cpu_count():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1
