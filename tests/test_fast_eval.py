"""The vectorised functional oracle (oracle/fast_eval.py) is pinned to the
reference's own `eval_program` (interpreter.py:223-245) before it is used
as a checker at sizes `eval_program` cannot reach: bit-identical results
on the reference's END_TO_END programs (test_lowering.py:27-88) and on the
programs of every benchmark config (plus the extension primitives), at
small sizes, with random inputs (CPU only)."""

import random

import numpy as np
import pytest

import fast_eval
from paper_2201_03611_b200 import gpu_rules, programs
from paper_2201_03611_b200._ref import interpreter, nat, types
from paper_2201_03611_b200.frontend import compile_program
from test_gpu_end_to_end import END_TO_END, PAIR_SUM, random_value

ArrayType = types.ArrayType


def _same(fast, ref):
    """Bit-identical f32 (NaN == NaN), exact ints, elementwise over nests."""
    a = np.asarray(fast_eval.to_plain(fast), dtype=np.float64 if _is_float(ref) else np.int64)
    b = np.asarray(interpreter.to_plain(ref), dtype=a.dtype)
    assert a.shape == b.shape
    if a.dtype == np.float64:
        fa, fb = a.astype(np.float32), b.astype(np.float32)
        assert np.array_equal(fa.view(np.uint32), fb.view(np.uint32)), (fa, fb)
    else:
        assert np.array_equal(a, b)


def _is_float(v):
    while isinstance(v, (list, tuple)):
        if not v:
            return True
        v = v[0]
    return isinstance(v, (float, np.floating))


def _inputs(program, nats, rng):
    out = []
    e = program
    from paper_2201_03611_b200._ref import expr

    DepLambda, Lambda = expr.DepLambda, expr.Lambda

    while True:
        if isinstance(e, DepLambda):
            e = e.body
        elif isinstance(e, Lambda):
            out.append(random_value(e.param.type, nats, rng))
            e = e.body
        else:
            return out


@pytest.mark.parametrize("case", END_TO_END, ids=[c[0] for c in END_TO_END])
def test_end_to_end_programs_bit_identical(case):
    name, source, nats = case
    c = compile_program(source, None, name=name)
    rng = random.Random(sum(map(ord, name)))
    for _ in range(10):
        inputs = _inputs(c.source_typed, nats, rng)
        _same(fast_eval.eval_program(c.source_typed, nats, inputs),
              interpreter.eval_program(c.source_typed, nats, inputs))


CONFIG_SIZES = {
    "dot": {"n": 64},
    "gemv": {"n": 8, "m": 12},
    "gemv_opt": {"n": 8, "m": 12, "s": 4},
    "conv": {"n": 6, "m": 7},
    "sgemm": {"n": 4, "m": 5, "k": 6},
    "nbody": {"n": 8},
    "sgemm_tiled": {"n": 4, "m": 5, "k": 64},
}


@pytest.mark.parametrize("key", sorted(CONFIG_SIZES))
def test_config_programs_bit_identical(key):
    c = programs.compile_config(key)
    nats = CONFIG_SIZES[key]
    rng = random.Random(len(key))
    for prog in (c.source_typed, c.lowered):  # before and after the strategy
        for _ in range(3):
            inputs = _inputs(prog, nats, rng)
            _same(fast_eval.eval_program(prog, nats, inputs), interpreter.eval_program(prog, nats, inputs))


@pytest.mark.parametrize("source,strategy,nats", [
    (programs.ASUM, programs.ASUM_STRATEGY, {"n": 33}),
    (PAIR_SUM, None, {}),
], ids=["asum", "pairSum"])
def test_more_programs_bit_identical(source, strategy, nats):
    c = compile_program(source, strategy)
    rng = random.Random(7)
    for _ in range(5):
        inputs = _inputs(c.source_typed, nats, rng)
        _same(fast_eval.eval_program(c.source_typed, nats, inputs),
              interpreter.eval_program(c.source_typed, nats, inputs))


def test_chunked_dot_schedule_bit_identical():
    # the GPU rewrite strategy's output (split-reduce), evaluated both ways
    c = compile_program(programs.DOT, gpu_rules.CHUNKED_REDUCE_STRATEGY, name="dotChunked")
    rng = random.Random(3)
    nats = {"n": 4096 * 3}
    inputs = _inputs(c.lowered, nats, rng)
    _same(fast_eval.eval_program(c.lowered, nats, inputs), interpreter.eval_program(c.lowered, nats, inputs))


def test_large_sizes_are_fast():
    # what eval_program cannot do in minutes: a 4096 x 4096 chunked dot and a 1024^2 gemv
    import time

    c = compile_program(programs.DOT, gpu_rules.CHUNKED_REDUCE_STRATEGY, name="dotChunked")
    a = np.random.default_rng(1).uniform(-1, 1, 1 << 24).astype(np.float32)
    b = np.random.default_rng(2).uniform(-1, 1, 1 << 24).astype(np.float32)
    t = time.perf_counter()
    out = fast_eval.to_numpy(fast_eval.eval_program(c.lowered, {"n": 1 << 24}, [a, b]))
    assert time.perf_counter() - t < 60
    # the same two-level order by hand: left folds of every chunk, then of the chunk sums
    chunks = np.zeros(4096, np.float32)
    pa, pb = a.reshape(4096, 4096), b.reshape(4096, 4096)
    for j in range(4096):
        chunks += pa[:, j] * pb[:, j]
    total = np.float32(0)
    for v in chunks:
        total = np.float32(total + v)
    assert out.view(np.uint32) == np.asarray(total).view(np.uint32)


@pytest.mark.parametrize("high,strategy_name,nats", [
    ("CONV_HIGH", "CONV_STRATEGY", {"n": 6, "m": 7}),
    ("NBODY_HIGH", "NBODY_STRATEGY", {"n": 8}),
])
def test_gpu_strategies_preserve_the_program_bit_for_bit(high, strategy_name, nats):
    """The conv and nbody strategies only fuse and lower (no reassociation):
    the rewritten program evaluates bit-identically to the high-level one."""
    c = compile_program(getattr(programs, high), getattr(gpu_rules, strategy_name))
    rng = random.Random(11)
    for _ in range(3):
        inputs = _inputs(c.source_typed, nats, rng)
        _same(fast_eval.eval_program(c.lowered, nats, inputs), interpreter.eval_program(c.source_typed, nats, inputs))


def test_sgemm_tiled_strategy_reassociates_k_into_tiles_only():
    """The sgemm strategy's one reassociation is the K fold in tiles of 32:
    the rewritten program equals sum over tiles of each tile's left fold."""
    c = compile_program(programs.SGEMM_HIGH, gpu_rules.SGEMM_TILED_STRATEGY)
    rng = np.random.default_rng(5)
    n, m, k = 4, 3, 96
    A = rng.uniform(-1, 1, (n, k)).astype(np.float32)
    B = rng.uniform(-1, 1, (k, m)).astype(np.float32)
    got = np.asarray(fast_eval.to_numpy(fast_eval.eval_program(c.lowered, {"n": n, "m": m, "k": k}, [A, B])),
                     np.float32).reshape(n, m)
    want = np.zeros((n, m), np.float32)
    for i in range(n):
        for j in range(m):
            total = np.float32(0)
            for t in range(k // 32):
                part = np.float32(0)
                for p in range(32 * t, 32 * t + 32):
                    part = np.float32(part + np.float32(A[i, p] * B[p, j]))
                total = np.float32(total + part)
            want[i, j] = total
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
