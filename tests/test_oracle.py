"""The oracle is pinned before it is trusted (CPU only).

* the C restatement (oracle/rise_oracle.c) reproduces, bit for bit, the
  golden vectors produced by the reference interpreter itself
  (tests/golden/make_golden.py -> eval_program, interpreter.py:238);
* the reference's own emitted C (oracle/_ref) reproduces the same vectors;
* at larger sizes the restatement and the reference's emitted C agree bit
  for bit (the reference C is bit-exact with eval_program, SURVEY.md §8 c).
"""

import json
from pathlib import Path

import numpy as np
import pytest

import oracle

GOLDEN = json.loads((Path(__file__).parent / "golden" / "oracle_golden.json").read_text())


def _arr(spec):
    a = np.array([int(h, 16) for h in spec["f32"]], dtype=np.uint32).view(np.float32)
    return a.reshape(spec["shape"]) if spec["shape"] else a.reshape(())


def _case(key):
    g = GOLDEN[key]
    return [_arr(i) for i in g["inputs"]], _arr(g["output"]), g["nats"]


def test_golden_file_covers_every_config():
    assert {"dot", "mv", "mv_opt", "sgemm_bt", "conv", "nbody", "kat_mv"} <= set(GOLDEN)


def test_oracle_dot_matches_reference_interpreter():
    (a, b), out, _ = _case("dot")
    assert oracle.dot(a, b).view(np.uint32) == out.view(np.uint32)


@pytest.mark.parametrize("key", ["mv", "mv_opt", "kat_mv"])
def test_oracle_mv_matches_reference_interpreter(key):
    (M, x), out, _ = _case(key)
    np.testing.assert_array_equal(oracle.mv(M, x).view(np.uint32), out.view(np.uint32))


def test_kat_mv_is_6_15():
    (M, x), out, _ = _case("kat_mv")
    assert out.tolist() == [6.0, 15.0] == GOLDEN["kat_mv"]["expect_plain"]


def test_oracle_sgemm_matches_reference_interpreter():
    (A, Bt), out, _ = _case("sgemm_bt")
    np.testing.assert_array_equal(oracle.sgemm_bt(A, Bt).view(np.uint32), out.view(np.uint32))


def test_oracle_conv_matches_extension_interpreter():
    (img, w), out, _ = _case("conv")
    np.testing.assert_array_equal(oracle.conv3x3(img, w).view(np.uint32), out.view(np.uint32))


def test_oracle_nbody_matches_extension_interpreter():
    (pos, vel, mass), out, _ = _case("nbody")
    np.testing.assert_array_equal(oracle.nbody(pos, vel, mass).view(np.uint32), out.view(np.uint32))


needs_ref = pytest.mark.skipif(oracle.ref_lib() is None, reason="oracle/_ref not built")


@needs_ref
def test_reference_emitted_c_matches_golden():
    (a, b), out, _ = _case("dot")
    assert oracle.ref_dot(a, b).view(np.uint32) == out.view(np.uint32)
    (M, x), out, nats = _case("mv_opt")
    np.testing.assert_array_equal(oracle.ref_mv(M, x, s=nats["s"]).view(np.uint32), out.view(np.uint32))
    (A, Bt), out, _ = _case("sgemm_bt")
    np.testing.assert_array_equal(oracle.ref_sgemm_bt(A, Bt).view(np.uint32), out.view(np.uint32))


@needs_ref
def test_restatement_equals_reference_c_at_size():
    a = oracle.rng_inputs(1, 1 << 20)
    b = oracle.rng_inputs(2, 1 << 20)
    assert oracle.dot(a, b) == oracle.ref_dot(a, b)
    M = oracle.rng_inputs(3, 512, 1024)
    x = oracle.rng_inputs(4, 1024)
    np.testing.assert_array_equal(oracle.mv(M, x), oracle.ref_mv(M, x))
    np.testing.assert_array_equal(oracle.mv(M, x), oracle.ref_mv(M, x, s=32))
    A = oracle.rng_inputs(5, 64, 96)
    Bt = oracle.rng_inputs(6, 48, 96)
    np.testing.assert_array_equal(oracle.sgemm_bt(A, Bt), oracle.ref_sgemm_bt(A, Bt))


@needs_ref
def test_reference_emitted_c_of_extension_programs_matches_golden():
    """conv / nbody through the reference's own emitter with the extension's
    emit_exp cases (extension.py §5) == the extension interpreter's golden
    vectors, bit for bit."""
    (img, w), out, _ = _case("conv")
    np.testing.assert_array_equal(oracle.ref_conv3x3(img, w).view(np.uint32), out.view(np.uint32))
    (pos, vel, mass), out, _ = _case("nbody")
    n = mass.size
    got = oracle.ref_nbody_block(pos, vel, mass, 0, n)
    np.testing.assert_array_equal(got.view(np.uint32), out.reshape(n, 3).view(np.uint32))


@needs_ref
def test_restatement_equals_reference_c_of_extension_programs_at_size():
    img = oracle.rng_inputs(3, 300, 260)
    w = oracle.rng_inputs(7, 3, 3)
    np.testing.assert_array_equal(oracle.conv3x3(img, w), oracle.ref_conv3x3(img, w))
    n = 2048
    pos = oracle.rng_inputs(5, n, 3)
    vel = oracle.rng_inputs(6, n, 3, low=-0.1, high=0.1)
    mass = oracle.rng_inputs(8, n, low=0.5, high=1.5)
    np.testing.assert_array_equal(oracle.nbody(pos, vel, mass, 100, 64),
                                  oracle.ref_nbody_block(pos, vel, mass, 100, 64))


@needs_ref
def test_reference_c_asum_is_the_sequential_fold():
    x = oracle.rng_inputs(9, 100003)
    want = np.add.accumulate(np.abs(x), dtype=np.float32)[-1]  # left fold from 0 (0 + a == a exactly)
    assert oracle.ref_asum(x).view(np.uint32) == np.float32(want).view(np.uint32)


@needs_ref
def test_reference_c_chunked_dot_is_the_chunked_fold():
    a = oracle.rng_inputs(1, 1 << 20)
    b = oracle.rng_inputs(2, 1 << 20)
    parts = np.array([oracle.dot(a[i:i + 4096], b[i:i + 4096]) for i in range(0, 1 << 20, 4096)], np.float32)
    want = oracle.dot(parts, np.ones_like(parts))
    assert np.float32(oracle.ref_dot_chunked(a, b)).view(np.uint32) == np.float32(want).view(np.uint32)


def test_left_fold_order_is_pinned():
    # interpreter.py:134-138: reduce is a left fold from init; 0.1+0.2+0.3 in
    # fp32 (test_interpreter.py:79-84) — the restatement does the same
    a = np.array([0.1, 0.2, 0.3], np.float32)
    one = np.ones(3, np.float32)
    expect = np.float32(np.float32(np.float32(0.0) + np.float32(0.1)) + np.float32(0.2)) + np.float32(0.3)
    assert oracle.dot(a, one) == expect


def test_error_bounds_are_sane():
    a = oracle.rng_inputs(1, 4096)
    b = oracle.rng_inputs(2, 4096)
    v64, s = oracle.dot_f64(a, b)
    # the reference's own sequential fp32 fold is inside the bound we grant
    # the reassociated GPU order
    assert abs(float(oracle.dot(a, b)) - v64) <= oracle.reassociated_dot_bound(4096, s, 4096)
