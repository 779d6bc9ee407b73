"""SURVEY §8 b: the back end is a drop-in — with its extension primitives
registered through the reference's seams and `integration.install()` putting
the sm100a target into the reference's own `codegen.emit`, CLI and
`cexec.run_emitted`, the REFERENCE's own test suite still passes (its
assertion that `emit(unit, "cuda")` raises included).  Runs the suite in a
subprocess from /root/reference (present in the build container only)."""

import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
REF_TESTS = Path("/root/reference/pkg/tests")

SCRIPT = f"""
import sys
sys.path.insert(0, {str(ROOT)!r})
import paper_2201_03611_b200  # the extension primitives, through the reference's seams
from paper_2201_03611_b200 import integration
integration.install()
import pytest
sys.exit(pytest.main(["-q", "-p", "no:cacheprovider", {str(REF_TESTS)!r}]))
"""


@pytest.mark.skipif(not REF_TESTS.is_dir(), reason="the reference's sources are not on this host")
def test_reference_suite_passes_with_the_backend_installed(tmp_path):
    r = subprocess.run([sys.executable, "-c", SCRIPT], cwd=tmp_path, capture_output=True, text=True, timeout=600)
    tail = (r.stdout + r.stderr)[-2000:]
    assert r.returncode == 0, tail
    assert " passed" in tail and "failed" not in tail
