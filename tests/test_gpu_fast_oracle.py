"""GPU results against the vectorised functional oracle (oracle/fast_eval.py,
pinned to the reference's `eval_program` by tests/test_fast_eval.py) at
sizes `eval_program` and `run_unit` cannot reach.  Every kernel here keeps
the program's order (the order-preserving templates, or the generic kernel
under reassociate=False), so the bar is bit-identity."""

import numpy as np
import pytest

import fast_eval
import oracle
from paper_2201_03611_b200 import compile_program, emit_cuda, gpu_rules, programs, run_cuda
from test_gpu_end_to_end import TILED_STAGES

pytestmark = pytest.mark.gpu


def _bits(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32)).view(np.uint32)


def _check(c, code, nats, inputs, program=None):
    got = run_cuda(code, c.unit, nats, inputs, as_numpy=True)
    want = fast_eval.to_numpy(fast_eval.eval_program(program or c.lowered, nats, inputs))
    assert np.array_equal(_bits(got).reshape(-1), _bits(want).reshape(-1))
    return code.plan["stages"]


def test_chunked_dot_full_size(gpu):
    c = compile_program(programs.DOT, gpu_rules.CHUNKED_REDUCE_STRATEGY, name="dotChunked")
    n = 1 << 24
    stages = _check(c, emit_cuda(c.unit, reassociate=False), {"n": n},
                    [oracle.rng_inputs(11, n), oracle.rng_inputs(12, n)])
    assert [s["kind"] for s in stages] == ["rowfold", "seqfold"]


@pytest.mark.parametrize("n,m,s", [(2048, 1024, 32), (1000, 516, 8), (8192, 1024, 32)])
def test_gemv_opt_schedule(gpu, n, m, s):
    cfg = programs.CONFIGS["gemv_opt"]
    c = compile_program(cfg["source"], cfg["strategy"], name="mv")
    _check(c, emit_cuda(c.unit), {"n": n, "m": m, "s": s}, [oracle.rng_inputs(13, n, m), oracle.rng_inputs(14, m)])


@pytest.mark.parametrize("n,m", [(1024, 768), (67, 1001)])
def test_conv_stencil(gpu, n, m):
    c = programs.compile_config("conv")
    w = np.array([[1, 2, 1], [2, 4, 2], [1, 2, 1]], np.float32) / np.float32(16)
    stages = _check(c, emit_cuda(c.unit), {"n": n, "m": m}, [oracle.rng_inputs(15, n, m), w])
    assert stages[0]["kind"] == "stencil2d"


def test_sgemm_in_program_order(gpu):
    c = programs.compile_config("sgemm")
    nats = {"n": 256, "m": 192, "k": 320}
    _check(c, emit_cuda(c.unit, reassociate=False), nats,
           [oracle.rng_inputs(16, 256, 320), oracle.rng_inputs(17, 192, 320)])


def test_nbody_in_program_order(gpu):
    c = programs.compile_config("nbody")
    n = 2048
    rng = np.random.default_rng(18)
    pos = rng.uniform(-1, 1, (n, 3)).astype(np.float32)
    vel = rng.uniform(-1, 1, (n, 3)).astype(np.float32)
    mass = rng.uniform(0.5, 1.5, n).astype(np.float32)
    _check(c, emit_cuda(c.unit, reassociate=False), {"n": n}, [pos, vel, mass])


@pytest.mark.parametrize("n,m", [(512, 1024), (3, 4)])
def test_tiled_stages_local_memory(gpu, n, m):
    c = compile_program(TILED_STAGES, None, name="tiledStages")
    _check(c, emit_cuda(c.unit), {"n": n, "m": m}, [oracle.rng_inputs(19, n, m)], program=c.source_typed)


def test_asum_in_program_order(gpu):
    # one flat left fold: the oracle steps it element by element (1 s at 2^16)
    c = compile_program(programs.ASUM, programs.ASUM_STRATEGY, name="asum")
    n = (1 << 16) + 3
    _check(c, emit_cuda(c.unit, reassociate=False), {"n": n}, [oracle.rng_inputs(20, n)])
