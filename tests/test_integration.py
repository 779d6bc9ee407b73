"""INTEGRATION.md §1 exercised from the reference side: with the shim
installed (paper_2201_03611_b200.integration), the reference's OWN entry
points — codegen.emit, the risec CLI, cexec.run_emitted — reach the sm100a
back end, and leave the reference's targets unchanged."""

import io
import json
from contextlib import redirect_stdout

import numpy as np
import pytest

from paper_2201_03611_b200 import emit_cuda, integration, programs
from paper_2201_03611_b200._ref import cexec, cli, codegen, errors

MV_SRC = programs.MV


@pytest.fixture()
def shim():
    integration.install()
    yield
    integration.uninstall()


def test_codegen_emit_dispatches_the_new_target(shim):
    unit = programs.compile_config("gemv").unit
    assert "sm100a" in codegen.TARGETS
    assert codegen.emit(unit, "sm100a") == emit_cuda(unit).text
    # the reference's own targets are untouched, and "cuda" is still rejected
    assert codegen.emit(unit, "opencl").startswith("__kernel\nvoid mvKernel(")
    with pytest.raises(errors.EmitError):
        codegen.emit(unit, "cuda")


def test_uninstall_restores_the_reference():
    integration.install()
    integration.uninstall()
    assert "sm100a" not in codegen.TARGETS
    with pytest.raises(errors.EmitError):
        codegen.emit(programs.compile_config("gemv").unit, "sm100a")


def test_risec_cli_emits_sm100a(shim, tmp_path):
    src = tmp_path / "mv.rise"
    src.write_text(MV_SRC)
    strat = tmp_path / "mv_opt.elv"
    strat.write_text(programs.MV_OPT_STRATEGY)
    out = tmp_path / "mv.cu"
    rc = cli.main([str(src), "--strategy", str(strat), "--target", "sm100a", "-o", str(out)])
    assert rc == 0
    text = out.read_text()
    assert text.startswith(integration.HEADER)
    c = programs.compile_config("gemv_opt")
    assert text == emit_cuda(c.unit).text  # the CLI's own front end reached the same unit


def test_run_emitted_keeps_the_reference_evaluator_for_its_text(shim):
    c = programs.compile_config("gemv")
    code = codegen.emit(c.unit, "opencl")
    got = cexec.run_emitted(code, c.unit, {"n": 2, "m": 3}, [[[1, 2, 3], [4, 5, 6]], [1, 1, 1]])
    assert [float(v) for v in got] == [6.0, 15.0]  # MV = [6, 15] (test_interpreter.py:37-40)


@pytest.mark.gpu
def test_run_emitted_runs_sm100a_text_on_the_gpu(shim, gpu):
    c = programs.compile_config("gemv")
    code = codegen.emit(c.unit, "sm100a")
    got = cexec.run_emitted(code, c.unit, {"n": 2, "m": 3}, [[[1, 2, 3], [4, 5, 6]], [1, 1, 1]])
    assert [float(v) for v in got] == [6.0, 15.0]
    # and at size, against the reference's own emitted C of the same unit
    import oracle

    rng = np.random.default_rng(2)
    M = rng.uniform(-1, 1, (300, 700)).astype(np.float32)
    x = rng.uniform(-1, 1, 700).astype(np.float32)
    got = np.asarray(cexec.run_emitted(code, c.unit, {"n": 300, "m": 700}, [M, x]), np.float32)
    np.testing.assert_array_equal(got, oracle.ref_mv(M, x))
