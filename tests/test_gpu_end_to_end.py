"""The reference's END_TO_END programs (test_lowering.py:27-88) and the MV
program on the GPU, compared with the reference's imperative interpreter
`run_unit` (interpreter.py:661, strict race checking) under the reference's
own comparison `values_close` (<= 4 ULP for f32, exact for i32;
interpreter.py:285-293) — the same oracle check the reference applies to
its emitted code (test_codegen.py:157-183), now for the sm100a target."""

import random

import numpy as np
import pytest

from paper_2201_03611_b200 import compile_program, emit_cuda, programs, run_cuda
from paper_2201_03611_b200._ref import interpreter, nat, types

ArrayType, ScalarType, TupleType = types.ArrayType, types.ScalarType, types.TupleType

pytestmark = pytest.mark.gpu

PAIR_SUM = """
def pairSum = fun(xs: Array[8, f32] =>
  xs |> iterate(3)(depFun((l: Nat) => fun(a: Array[l * 2, f32] =>
    a |> split(2) |> mapSeq(fun(p =>
      p |> reduceSeq(Private)(fun(acc, v => acc + v))(0.0f) )) ))) )
"""

TILED_STAGES = """
def f = fun(z: f32 => z * 2.0f)
def g = fun(z: f32 => z + 1.0f)
def stages = depFun((n: Nat, m: Nat) =>
  fun(M: Array[n, Array[m, f32]] =>
    M |> mapWorkGroup(fun(row =>
      row |> mapLocal(f) |> toMem(Private) |> mapLocal(g)) )))
"""

# (name, source, sizes) — test_lowering.py:27-88
END_TO_END = [
    ("scaleSeq", "fun(xs: Array[6, f32] => xs |> mapSeq(fun(v => v * 2.0f)))", {}),
    ("mapMapToMem", "fun(xs: Array[8, f32] => xs |> mapSeq(fun(v => v + 1.0f)) |> toMem(Private) |> mapSeq(fun(v => v * 3.0f)))", {}),
    ("dotProduct", "fun(a: Array[5, f32] => fun(b: Array[5, f32] => zip(a)(b) |> mapSeq(fun(p => fst(p) * snd(p))) |> toMem(Private) |> reduceSeq(Private)(fun(acc, v => acc + v))(0.0f)))", {}),
    ("sumOfSquares", "fun(xs: Array[7, i32] => xs |> reduceSeq(Private)(fun(acc, v => acc + v * v))(0))", {}),
    ("rowSums", "fun(M: Array[3, Array[4, f32]] => M |> mapSeq(fun(row => row |> reduceSeq(Private)(fun(a, v => a + v))(0.0f))))", {}),
    ("chunkedScale", "fun(xs: Array[12, f32] => xs |> split(4) |> mapSeq(fun(c => c |> mapSeq(fun(v => v * 0.5f)))) |> join)", {}),
    ("zipAdd", "fun(a: Array[6, i32] => fun(b: Array[6, i32] => zip(a)(b) |> mapSeq(fun(p => fst(p) + snd(p)))))", {}),
    ("globalScale", "depFun((n: Nat) => fun(xs: Array[n, f32] => xs |> mapGlobal(fun(v => v * 4.0f))))", {"n": 10}),
    ("tiledStages", TILED_STAGES, {"n": 3, "m": 4}),
    ("pairSum", PAIR_SUM, {}),
]


def random_value(dtype, nat_env, rng):
    # conftest.py:57-71 of the reference suite
    if isinstance(dtype, ArrayType):
        size = nat.evaluate(dtype.size, nat_env)
        return [random_value(dtype.elem, nat_env, rng) for _ in range(size)]
    if isinstance(dtype, TupleType):
        return [random_value(dtype.fst, nat_env, rng), random_value(dtype.snd, nat_env, rng)]
    if isinstance(dtype, ScalarType):
        if dtype.name == "f32":
            return round(rng.uniform(-4.0, 4.0), 3)
        if dtype.name == "i32":
            return rng.randint(-50, 50)
    raise AssertionError(dtype)


@pytest.mark.parametrize("case", END_TO_END, ids=[c[0] for c in END_TO_END])
def test_end_to_end_program_matches_run_unit(gpu, case):
    name, source, nats = case
    c = compile_program(source, None, name=name)
    code = emit_cuda(c.unit)
    rng = random.Random(sum(map(ord, name)))  # PYTHONHASHSEED-independent (SURVEY.md §4 flakiness note)
    for _ in range(20):
        inputs = [random_value(dt, nats, rng) for _v, dt in c.unit.inputs]
        got = run_cuda(code, c.unit, nats, inputs)
        ref = interpreter.run_unit(c.unit, nats, inputs, strict=True)
        assert interpreter.values_close(got, ref), (name, inputs, got, ref)


def test_pair_sum_known_answer(gpu):
    # test_interpreter.py:67-76 / test_codegen.py:137-148: [1..8] -> 36
    c = compile_program(PAIR_SUM, None, name="pairSum")
    out = run_cuda(emit_cuda(c.unit), c.unit, {}, [[1, 2, 3, 4, 5, 6, 7, 8]])
    assert interpreter.values_close(out, [np.float32(36.0)])


@pytest.mark.parametrize("strategy", [programs.MV_GLOBAL_STRATEGY, programs.MV_OPT_STRATEGY])
def test_mv_matches_run_unit(gpu, strategy):
    c = compile_program(programs.MV, strategy, name="mv")
    code = emit_cuda(c.unit)
    nats = {"n": 4, "m": 8, "s": 2}
    rng = random.Random(1)
    for _ in range(20):
        inputs = [random_value(dt, nats, rng) for _v, dt in c.unit.inputs]
        got = run_cuda(code, c.unit, nats, inputs)
        ref = interpreter.run_unit(c.unit, nats, inputs, strict=True)
        assert interpreter.values_close(got, ref)


def test_global_toMem_between_parallel_stages(gpu):
    # SURVEY §8 a (iii): two kernels with a runtime-allocated Global temporary
    src = ("depFun((n: Nat) => fun(xs: Array[n, f32] => xs |> mapGlobal(fun(v => v * 2.0f)) "
           "|> toMem(Global) |> mapGlobal(fun(v => v + 1.0f))))")
    c = compile_program(src, None, name="twoStage")
    code = emit_cuda(c.unit)
    xs = [float(i) for i in range(1000)]
    got = run_cuda(code, c.unit, {"n": 1000}, [xs])
    assert interpreter.values_close(got, interpreter.run_unit(c.unit, {"n": 1000}, [xs]))


def test_local_memory_with_barriers(gpu):
    # SURVEY §8 a (ii): toMem(Local) between mapLocal stages
    src = ("depFun((n: Nat, m: Nat) => fun(M: Array[n, Array[m, f32]] => M |> mapWorkGroup(fun(row => "
           "row |> mapLocal(fun(z => z * 2.0f)) |> toMem(Local) |> mapLocal(fun(z => z + 1.0f))))))")
    c = compile_program(src, None, name="localStages")
    code = emit_cuda(c.unit)
    rng = random.Random(3)
    nats = {"n": 37, "m": 300}
    M = [[round(rng.uniform(-4, 4), 3) for _ in range(300)] for _ in range(37)]
    got = run_cuda(code, c.unit, nats, [M])
    assert interpreter.values_close(got, interpreter.run_unit(c.unit, nats, [M]))


def test_left_fold_known_answer(gpu):
    # test_interpreter.py:55-57: reduce is a left fold from init: [1,2,3,4] with a - b from 0 -> -10
    c = compile_program("fun(xs: Array[4, f32] => xs |> reduce(fun(a, b => a - b))(0.0f))",
                        "toReduceSeq @ every(isReduce)", name="leftFold")
    out = run_cuda(emit_cuda(c.unit), c.unit, {}, [[1.0, 2.0, 3.0, 4.0]])
    assert interpreter.values_close(out, np.float32(-10.0))


def test_fuse_reduce_map_known_answer(gpu):
    # test_rules.py:212-216: map(v * v) >> reduce(add)(0) fused -> 14 on [1, 2, 3]
    c = compile_program("fun(xs: Array[3, i32] => xs |> map(fun(v => v * v)) |> reduce(add)(0))",
                        "fuseReduceMap @ every(isReduce) ; toReduceSeq @ every(isReduce)", name="sumSq")
    out = run_cuda(emit_cuda(c.unit), c.unit, {}, [[1, 2, 3]])
    assert int(np.asarray(out).reshape(-1)[0]) == 14


ITERATE_BIG = """
def pairSum = depFun((n: Nat) => fun(xs: Array[8 * n, f32] =>
  xs |> iterate(3)(depFun((l: Nat) => fun(a: Array[l * 2, f32] =>
    a |> split(2) |> mapGlobal(fun(p =>
      p |> reduceSeq(Private)(fun(acc, v => acc + v))(0.0f) )) ))) ))
"""


@pytest.mark.parametrize("n", [1, 1000, 1 << 20])
def test_iterate_on_the_whole_gpu(gpu, n):
    """iterate(3) of a parallel pairwise sum: the `iterate` template keeps
    the ping-pong buffers in global memory and separates the steps with a
    grid-wide barrier of a cooperative launch, so sizes far beyond shared
    memory run; bit-exact with the program's own order."""
    from paper_2201_03611_b200.run import Executable

    c = compile_program(ITERATE_BIG, None, name="pairSum")
    code = emit_cuda(c.unit)
    assert Executable(code, {"n": n}).template_kinds == ["iterate"]
    xs = np.random.default_rng(n).uniform(-1, 1, 8 * n).astype(np.float32)
    got = run_cuda(code, c.unit, {"n": n}, [xs], as_numpy=True)
    want = xs
    for _ in range(3):  # each step: (0 + a[2g]) + a[2g + 1]
        want = ((np.float32(0) + want[0::2]) + want[1::2]).astype(np.float32)
    np.testing.assert_array_equal(got, want)
    if n <= 1000:  # and the reference's imperative interpreter agrees
        ref = interpreter.run_unit(c.unit, {"n": n}, [[np.float32(v) for v in xs]])
        np.testing.assert_array_equal(np.asarray(ref, np.float32), want)
