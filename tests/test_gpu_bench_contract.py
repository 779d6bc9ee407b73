"""bench.py keeps the driver's JSON-line contract (one line on stdout with
the metric, the timing, the roofline, the end-to-end figure, clocks and the
launch count, plus `per_config` for every BASELINE config) — short runs on
the GPU, and `--gpus 2` really runs two ranks (sharing the one GPU here)."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent


def _line(out):
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [x for x in out.stdout.strip().splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def _check_entry(d):
    assert d["value"] > 0 and d["ms_per_step"] > 0
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(d["roofline"])
    assert {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= set(d["e2e"])
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and "workload" in d["config"]
    assert d["gpu_launches"] >= 3


def test_bench_prints_one_contract_line_with_every_config(gpu):
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--steps", "3", "--warmup", "3",
                          "--no-cpu-baseline"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    d = _line(out)
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "roofline", "clocks"):
        assert key in d, key
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    _check_entry(d)
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert set(d["per_config"]) == {"dot", "gemv", "conv", "sgemm_tiled", "nbody"}
    for key, entry in d["per_config"].items():
        _check_entry(entry)
        assert entry["config"]["workload"].startswith(key)
        # build times outside the timed region; individually timed steps where the L2 is flushed
        assert {"emit_s", "nvrtc_and_load_s"} <= set(entry["impl_detail"]["build"])
        if key in ("sgemm_tiled", "nbody"):
            st = entry["impl_detail"]["step_ms"]
            assert 0 < st["best"] <= st["median"] <= st["worst"]
    assert d["per_config"]["gemv"]["value"] == d["value"]
    assert "peak_note" in d["roofline"]  # the HBM peak is a copy rate; read-only streams may exceed it


def test_bench_gpus_2_runs_two_ranks(gpu):
    env = dict(os.environ, RISE_BENCH_SHARED_GPU="1", RISE_DIST_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3",
                          "--configs", "dot,conv,sgemm_tiled,nbody"], cwd=ROOT, capture_output=True, text=True,
                         timeout=900, env=env)
    d = _line(out)
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["sizes"] == {"n": 8192, "m": 8192}  # the BASELINE shape, split over the ranks
    assert d["impl_detail"]["rank_sizes"] == {"n": 4096, "m": 8192}
    assert "with_collective" in d
    for key, entry in d["per_config"].items():
        _check_entry(entry)
    assert d["per_config"]["sgemm_tiled"]["impl_detail"]["rank_sizes"]["n"] == 2048
    assert d["per_config"]["dot"]["impl_detail"]["rank_sizes"]["n"] == 1 << 23


def test_bench_refuses_more_gpus_than_visible(gpu):
    import torch

    n = torch.cuda.device_count() + 1
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.pop("RISE_BENCH_SHARED_GPU", None)
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", str(n), "--steps", "3"], cwd=ROOT,
                         capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode != 0 and "CUDA device" in out.stderr
