"""bench.py's host logic on CPU: the strong-scaled decomposition of every
BASELINE config covers the config's global input exactly once, and both
arms describe a config with the same `config` object."""

import importlib.util
import json
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


def _bench():
    spec = importlib.util.spec_from_file_location("rise_bench", ROOT / "bench.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


class _Small:
    """Shrink a workload class to test sizes (same decomposition code)."""

    def __init__(self, cls, **sizes):
        self.cls, self.sizes = cls, sizes

    def make(self, rank, world):
        wl = self.cls(rank, world, "strong")
        for k, v in self.sizes.items():
            setattr(wl, k, v)
        return wl


@pytest.mark.parametrize("world", [2, 4, 8])
def test_strong_bands_cover_the_global_input(world):
    bench = _bench()
    cases = {
        "gemv": _Small(bench.Gemv, n=64, m=32),
        "dot": _Small(bench.Dot, n=4096),
        "conv": _Small(bench.Conv, n=64, m=40),
        "sgemm": _Small(bench.Sgemm, n=64, m=32, k=16),
        "nbody": _Small(bench.Nbody, n=64),
    }
    for key, small in cases.items():
        whole = small.make(0, 1).global_inputs()
        parts = [small.make(r, world).local() for r in range(world)]
        if key in ("gemv", "sgemm"):
            got = np.concatenate([p[2][0] for p in parts])
            assert np.array_equal(got, whole[0]), key
            assert all(np.array_equal(p[2][1], whole[1]) for p in parts), key  # replicated operand
            assert sum(p[1]["n"] for p in parts) == whole[0].shape[0]
        elif key == "dot":
            for k in range(2):
                assert np.array_equal(np.concatenate([p[2][k] for p in parts]), whole[k])
        elif key == "conv":
            # fused halo: each band is exactly its rows, read by neighbours in place
            got = np.concatenate([p[2][0] for p in parts])
            assert np.array_equal(got, whole[0])
            assert sum(p[1]["n"] for p in parts) == whole[0].shape[0]
        else:
            t = whole[0].shape[0] // world
            got = np.concatenate([p[2][0] for p in parts])
            assert np.array_equal(got, whole[0])
            assert all(p[1] == {"t": t, "n": whole[0].shape[0]} for p in parts)


def test_both_arms_share_the_config_object():
    bench = _bench()
    for key in bench.PER_CONFIG:
        for world in (1, 2, 8):
            a = bench.config_of(bench.WORKLOADS[key](0, world), world)
            b = bench.config_of(bench.WORKLOADS[key](0, world), world)
            assert a == b and a["sizes"] and a["n_gpus"] == world


def test_reference_arm_per_config_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--configs", "dot,gemv,conv",
                          "--steps", "1", "--warmup", "3"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [x for x in out.stdout.strip().splitlines() if x.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and set(d["per_config"]) == {"dot", "gemv", "conv"}
    for key, r in d["per_config"].items():
        # one execution per step: value and ms_per_step agree
        assert r["value"] == pytest.approx(bench_work(key) / (r["ms_per_step"] * 1e-3) / 1e9, rel=2e-3)
        assert r["config"]["sizes"] and r["cpu_baseline"]["cores"] >= 1
    assert d["config"] == d["per_config"]["gemv"]["config"]


def bench_work(key):
    bench = _bench()
    return bench.WORKLOADS[key](0, 1).work()


def test_each_workload_compiles_its_own_program():
    """Every bench workload emits the unit of the program it names (the C4
    entry is the tiled program, not the flat one)."""
    bench = _bench()
    want = {"gemv": "mv", "gemv_opt": "mv", "dot": "dot", "dot_chunked": "dotChunked", "conv": "conv",
            "sgemm": "sgemm", "sgemm_nn": "sgemm", "sgemm_tiled": "sgemmTiled", "nbody": "nbody"}
    for key, unit in want.items():
        compiled, _nats = bench.WORKLOADS[key](0, 1).compile()
        assert compiled.unit.name == unit, key


def test_secondary_baseline_is_the_reference_interpreter():
    """cpu_baseline.secondary (SURVEY §8 d): the reference's pure-Python
    eval_program on each config's program at its reduced size — finishes in
    seconds, one core, a positive rate in the config's unit."""
    bench = _bench()
    for key in bench.PER_CONFIG:
        wl = bench.WORKLOADS[key]()
        sec = bench.python_reference(wl)
        assert sec["cores"] == 1 and sec["kind"] == "reference" and sec["unit"] == wl.metric_unit
        assert sec["value"] > 0 and sec["seconds"] < 30
        assert "eval_program" in sec["sample"]
