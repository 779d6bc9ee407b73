#!/usr/bin/env python3
"""Benchmark of the RISE/Shine sm100a back end (the BASELINE.json metric).

One step = one execution of the hot path — the RISE program's kernel(s),
emitted by `emit_cuda` from the ImperativeUnit the reference front end
produces — over one batch of synthetic, seeded input already resident in
HBM.  The headline is BASELINE.json configs[1], gemv fp32 8192x8192
(`mv.rise` + the toMapGlobal strategy); the same JSON line carries
`per_config`, every BASELINE config (C1 dot, C2 gemv, C3 conv, C4 sgemm,
C5 nbody; C4 as the tiled program BASELINE names) measured the same way, each with its roofline, its full-size CPU
baseline (the reference's emitted C/OpenMP on this host) and its e2e figure.

`--gpus N` runs N ranks, one per GPU: without torchrun's environment the
script launches them itself (`torch.distributed.run`, 127.0.0.1).  Scaling
is STRONG by default — every config keeps its BASELINE shape and the ranks
split it (row bands of M / A / the image, chunks of the dot, target blocks
of the bodies); `--scaling weak` gives every rank a full-size part of an
N-times larger problem instead.

Prints ONE JSON line (rank 0).  Timing: W warm-up steps; K timed steps
bracketed by barrier + synchronize, timed with CUDA events on the launching
stream, max over ranks.  HBM-bound configs use inputs larger than L2: R
input sets (>= 512 MiB, 4x the L2, in total) round robin, the K steps back
to back between two events; compute-bound ones flush the L2 (256 MiB write
+ read) before every step, outside that step's events.  `e2e` repeats the
step through the public host-buffer path (pinned H2D, kernels, D2H).
`--impl reference` times the reference's own CPU implementation (its
emitted C/OpenMP, oracle/_ref) on this host's cores instead.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import socket
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))  # checker / CPU-baseline legs only

L2_FLUSH_BYTES = 256 << 20
L2_BYTES = 126 << 20  # B200 L2
ROTATE_BYTES = 512 << 20  # input sets used round robin cover >= 4x L2
FP32_SIMT_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12  # derived, BASELINE.md §2
TF32_DENSE_TFLOPS = 1100.0  # B200_PROFILING.md fallback (MEASURED_PEAKS has no TF32 entry)
HEADLINE = "gemv"
# BASELINE.json configs[0..4]; C4 is the tiled split / transpose / toMem(Local) lowering it names
PER_CONFIG = ("dot", "gemv", "conv", "sgemm_tiled", "nbody")
METRIC = "per-benchmark GFLOP/s or GB/s vs B200 roofline at 1/2/4/8 GPUs vs CPU ref"


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "source": "measured (MEASURED_PEAKS.json)",
                "sm_max_mhz": d.get("sm_max_mhz", 1965.0), "bf16_tflops": d.get("bf16_tflops")}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)", "sm_max_mhz": 1965.0, "bf16_tflops": 1590.0}


# ---------------------------------------------------------------------------
# workloads: program, sizes, synthetic inputs, algorithmic work, decomposition


class Workload:
    """One BASELINE config.  `global_inputs()` is the config's seeded input
    (the same on every rank); `local()` is this rank's part of it: the
    program, sizes, host arrays and emission options of the rank's step."""

    key = ""
    config_index = 0
    emit_kwargs: dict = {}
    compute_bound = False

    def __init__(self, rank=0, world=1, scaling="strong"):
        self.rank, self.world, self.scaling = rank, world, scaling
        self.emit_kwargs = dict(type(self).emit_kwargs)

    def seed(self):
        # strong scaling splits ONE global problem; weak gives each rank its own
        return self.config_index + (1000 * self.rank if self.scaling == "weak" else 0)

    def total_work(self):
        return self.work() * (self.world if self.scaling == "weak" else 1)

    def local(self):
        compiled, nats = self.compile()
        host = self.global_inputs()
        if self.world == 1 or self.scaling == "weak":
            return self.weak_local(compiled, nats, host)
        return self.strong_local(compiled, nats, host)

    def weak_local(self, compiled, nats, host):
        return compiled, nats, host

    def band(self, total):
        from paper_2201_03611_b200.shard import row_band

        start, count = row_band(total, self.world, self.rank)
        return start, start + count

    def parallelism(self):
        raise NotImplementedError

    def cpu_alt_fn(self, host):
        return None  # a second reference CPU implementation of the same config, where one exists


class Gemv(Workload):
    key = "gemv"
    program = "mv.rise + toMapGlobal strategy (BASELINE.md §4 C2)"
    config_index = 2
    n = m = 8192
    metric_unit = "GB/s"
    bound = "hbm"

    def sizes(self):
        return {"n": self.n, "m": self.m}

    def compile(self):
        from paper_2201_03611_b200 import programs

        return programs.compile_config(self.key), self.sizes()

    def global_inputs(self):
        rng = np.random.default_rng(self.seed())
        M = rng.uniform(-1, 1, (self.n, self.m)).astype(np.float32)
        x = rng.uniform(-1, 1, self.m).astype(np.float32)
        return [M, x]

    def strong_local(self, compiled, nats, host):
        M, x = host
        r0, r1 = self.band(self.n)
        return compiled, dict(nats, n=r1 - r0), [np.ascontiguousarray(M[r0:r1]), x]

    def work(self):  # algorithmic bytes per step (SURVEY.md §8 d)
        return 4.0 * (self.n * self.m + self.m + self.n)

    def cpu_fn(self, host):
        import oracle

        M, x = host
        return (lambda: oracle.ref_mv(M, x)), oracle.threads(), (
            f"full {self.n}x{self.m} gemv, the reference's emitted OpenMP C (mv.rise + toMapGlobal, oracle/_ref)")

    def parallelism(self):
        if self.scaling == "weak":
            return f"weak: rank r owns an 8192-row band of a ({self.world}x8192) x 8192 matrix, x replicated, y sharded"
        return f"strong: 8192/{self.world} rows of M per rank, x replicated, y sharded (with_collective: y all-gathered)"


class GemvOpt(Gemv):
    key = "gemv_opt"
    program = "mv.rise + the paper's Listing-3 strategy (mv_opt.elv), s = 32"

    def sizes(self):
        return {"n": self.n, "m": self.m, "s": 32}


class Dot(Workload):
    key = "dot"
    program = "zip |> map(*) |> reduce(add) + fuseReduceMap;toReduceSeq (BASELINE.md §4 C1)"
    config_index = 1
    n = 1 << 24
    metric_unit = "GB/s"
    bound = "hbm"

    def sizes(self):
        return {"n": self.n}

    def compile(self):
        from paper_2201_03611_b200 import programs

        return programs.compile_config(self.key), self.sizes()

    def global_inputs(self):
        rng = np.random.default_rng(self.seed())
        return [rng.uniform(-1, 1, self.n).astype(np.float32), rng.uniform(-1, 1, self.n).astype(np.float32)]

    def _peer(self, compiled, nats, host):
        if _dot_peer():
            # the fused variant: each rank's reduce kernel publishes its total into
            # every rank's exchange slots (peer memory) and folds them in rank order
            self.emit_kwargs = {"peer_ranks": self.world}
        return compiled, nats, host

    def weak_local(self, compiled, nats, host):
        if self.world > 1:
            return self._peer(compiled, nats, host)
        return compiled, nats, host

    def strong_local(self, compiled, nats, host):
        a, b = host
        c0, c1 = self.band(self.n)
        return self._peer(compiled, dict(nats, n=c1 - c0), [a[c0:c1].copy(), b[c0:c1].copy()])

    def work(self):
        return 8.0 * self.n + 4

    def cpu_fn(self, host):
        import oracle

        a, b = host
        return (lambda: oracle.ref_dot(a, b)), 1, (
            "full 2^24 dot, the reference's emitted C (a sequential left fold: the reference lowers reduce to one "
            "loop, 1 thread)")

    def cpu_alt_fn(self, host):
        """beside C1's sequential fold, the reference's own
        OpenMP emission of the chunked schedule on all cores."""
        import oracle

        if oracle.ref_lib() is None:
            return None
        a, b = host
        return (lambda: oracle.ref_dot_chunked(a, b)), oracle.threads(), (
            "full 2^24 dot, the reference's emitted OpenMP C of the chunked schedule (dot + "
            "gpu_rules.CHUNKED_REDUCE_STRATEGY), all cores")

    def parallelism(self):
        how = ("the reduce kernel publishes its total into every rank's slots over NVLink (peer memory) and folds "
               "the totals in rank order (exchange fused into the kernel)" if _dot_peer() else
               "partials all-gathered (rs_allgather, NCCL) and folded in rank order")
        if self.scaling == "weak":
            return "weak: rank r owns a 2^24 chunk; " + how
        return f"strong: 2^24/{self.world} contiguous elements per rank; " + how


class DotChunked(Dot):
    cpu_alt_fn = Workload.cpu_alt_fn

    key = "dot_chunked"
    program = ("C1 (dot.rise) + the chunked-reduce strategy (gpu_rules.CHUNKED_REDUCE_STRATEGY: splitReduce(4096), "
               "...) -> split(4096) |> mapGlobal(reduceSeq) |> toMem(Global) |> reduceSeq (bit-exact)")
    emit_kwargs = {"reassociate": False}

    def compile(self):
        from paper_2201_03611_b200 import compile_program, gpu_rules, programs

        c = compile_program(programs.DOT, gpu_rules.CHUNKED_REDUCE_STRATEGY, name="dotChunked")
        return c, self.sizes()

    def _peer(self, compiled, nats, host):
        return compiled, nats, host  # partials all-gathered (NCCL), rank-order fold

    def cpu_fn(self, host):
        import oracle

        if oracle.ref_lib() is None:
            return super().cpu_fn(host)
        a, b = host
        return (lambda: oracle.ref_dot_chunked(a, b)), oracle.threads(), (
            "full 2^24 dot, the reference's emitted OpenMP C of the same chunked schedule (chunks in parallel, then "
            "the fold of the partials)")

    def parallelism(self):
        return f"{self.scaling}: per-rank chunk partials all-gathered (rs_allgather, NCCL), rank-order fold"


class Conv(Workload):
    key = "conv"
    program = "padClamp2D + slide2D + map/reduce 3x3 (programs.CONV)"
    config_index = 3
    n = m = 8192
    metric_unit = "GB/s"
    bound = "hbm"

    def sizes(self):
        return {"n": self.n, "m": self.m}

    def compile(self):
        from paper_2201_03611_b200 import programs

        return programs.compile_config(self.key), self.sizes()

    def global_inputs(self):
        rng = np.random.default_rng(self.seed())
        img = rng.uniform(-1, 1, (self.n, self.m)).astype(np.float32)
        w = (np.array([[1, 2, 1], [2, 4, 2], [1, 2, 1]], np.float32) / 16).astype(np.float32)
        return [img, w]

    def _banded(self, compiled, nats, band, w):
        if _conv_fused_halo():
            # the fused variant: the stencil kernel reads its neighbours' edge rows
            # in place (peer pointers), so the band is exactly this rank's rows
            self.emit_kwargs = {"peer_halo": True}
            return compiled, dict(nats, n=band.shape[0]), [band, w]
        local = np.empty((band.shape[0] + 2, band.shape[1]), np.float32)
        local[1:-1] = band
        local[0], local[-1] = band[0], band[-1]
        return compiled, dict(nats, n=band.shape[0] + 2), [local, w]

    def weak_local(self, compiled, nats, host):
        if self.world > 1:
            return self._banded(compiled, nats, host[0], host[1])
        return compiled, nats, host

    def strong_local(self, compiled, nats, host):
        img, w = host
        r0, r1 = self.band(self.n)
        return self._banded(compiled, nats, np.ascontiguousarray(img[r0:r1]), w)

    def work(self):
        return 4.0 * (2 * self.n * self.m + 9)

    def cpu_fn(self, host):
        import oracle

        img, w = host
        if oracle.ref_lib() is not None:
            return (lambda: oracle.ref_conv3x3(img, w)), oracle.threads(), (
                f"full {self.n}x{self.m} conv, the reference's emitted OpenMP C for programs.CONV (extension "
                "primitives through the emitter's seams, oracle/_ref)")
        return (lambda: oracle.conv3x3(img, w)), oracle.threads(), "C restatement (oracle/rise_oracle.c), OpenMP"

    def parallelism(self):
        how = ("the stencil kernel reads the neighbours' edge rows in place over NVLink (peer pointers, halo "
               "exchange fused into the border-tile staging)" if _conv_fused_halo() else
               "halo rows pulled from the neighbours' bands over NVLink (rs_halo_exchange, CUDA IPC) per step")
        if self.scaling == "weak":
            return "weak: rank r owns an 8192-row band; " + how
        return f"strong: 8192/{self.world} image rows per rank; " + how


class Sgemm(Workload):
    key = "sgemm"
    program = "A |> mapGlobal(arow => Bt |> mapGlobal(brow => zip |> reduceSeq)) (programs.SGEMM_BT)"
    config_index = 4
    n = m = k = 4096
    metric_unit = "GFLOP/s"
    bound = "tensor"
    compute_bound = True

    def sizes(self):
        return {"n": self.n, "m": self.m, "k": self.k}

    def compile(self):
        from paper_2201_03611_b200 import programs

        return programs.compile_config(self.key), self.sizes()

    def global_inputs(self):
        rng = np.random.default_rng(self.seed())
        A = rng.uniform(-1, 1, (self.n, self.k)).astype(np.float32)
        Bt = rng.uniform(-1, 1, (self.m, self.k)).astype(np.float32)
        return [A, Bt]

    def strong_local(self, compiled, nats, host):
        A, B = host
        r0, r1 = self.band(self.n)
        return compiled, dict(nats, n=r1 - r0), [np.ascontiguousarray(A[r0:r1]), B]

    def work(self):
        return 2.0 * self.n * self.m * self.k

    def cpu_fn(self, host):
        import oracle

        A, Bt = host
        return (lambda: oracle.ref_sgemm_bt(A, Bt)), oracle.threads(), (
            "full 4096^3 sgemm, the reference's emitted OpenMP C (oracle/_ref, sgemmBt: rows in parallel, each "
            "output a sequential k fold)")

    def parallelism(self):
        if self.scaling == "weak":
            return f"weak: rank r owns a 4096-row block of A ({self.world}x4096 rows), B replicated"
        return (f"strong: 4096/{self.world} rows of A per rank, B replicated, C row blocks (with_collective: B "
                "all-gathered from 1/N row blocks before the GEMM)")


class SgemmNN(Sgemm):
    key = "sgemm_nn"
    program = ("A |> mapGlobal(arow => transpose(B) |> mapGlobal(bcol => zip |> reduceSeq)) (programs.SGEMM; "
               "B row-major, MN-major tensor-core operand)")

    def compile(self):
        from paper_2201_03611_b200 import compile_program, programs

        return compile_program(programs.SGEMM, None, name="sgemm"), self.sizes()

    def global_inputs(self):
        A, Bt = super().global_inputs()
        return [A, np.ascontiguousarray(Bt.T)]

    def cpu_fn(self, host):
        A, B = host
        return super().cpu_fn([A, np.ascontiguousarray(B.T)])  # the reference C takes Bt


class SgemmTiled(SgemmNN):
    key = "sgemm_tiled"
    program = ("the tiled C4 program (programs.SGEMM_TILED: split / transpose / toMem(Local) under mapWorkGroup / "
               "mapLocal, K tiles) -> the tcgen05 3xTF32 template")

    def compile(self):
        from paper_2201_03611_b200 import programs

        return programs.compile_config(self.key), self.sizes()


class Nbody(Workload):
    key = "nbody"
    program = "all-pairs map/reduce + Euler velocity step (programs.NBODY)"
    config_index = 5
    n = int(os.environ.get("RISE_NBODY_N", "131072"))  # (probes only; the config is 131072)
    metric_unit = "GFLOP/s"
    bound = "fp32-simt"
    compute_bound = True

    def sizes(self):
        return {"n": self.n}

    def compile(self):
        from paper_2201_03611_b200 import programs

        return programs.compile_config(self.key), self.sizes()

    def global_inputs(self):
        rng = np.random.default_rng(self.config_index)
        pos = rng.uniform(-1, 1, (self.n, 3)).astype(np.float32)
        vel = np.zeros((self.n, 3), np.float32)
        mass = rng.uniform(0.5, 1.5, self.n).astype(np.float32)
        return [pos, vel, mass]

    def total_work(self):
        return self.work()  # always one global system (target blocks)

    def local(self):
        compiled, nats = self.compile()
        host = self.global_inputs()
        if self.world == 1:
            return compiled, nats, host
        from paper_2201_03611_b200 import compile_program, programs

        pos, vel, mass = host
        n = self.n
        if n % self.world:
            raise SystemExit(f"nbody: {n} bodies do not split over {self.world} ranks")
        t = n // self.world
        t0 = self.rank * t
        c = compile_program(programs.NBODY_SHARD, None, name="nbodyShard")
        if _nbody_peer():
            # the fused variant: each rank holds only its block; the kernel
            # reads every other block in place over NVLink (peer pointers)
            self.emit_kwargs = {"peer_ranks": self.world}
            blk = pos[t0:t0 + t]
            return c, {"t": t, "n": n}, [blk, vel[t0:t0 + t], blk, mass[t0:t0 + t]]
        return c, {"t": t, "n": n}, [pos[t0:t0 + t], vel[t0:t0 + t], pos, mass]

    def work(self):
        return 20.0 * self.n * self.n

    def cpu_fn(self, host):
        import oracle

        pos, vel, mass = host
        if oracle.ref_lib() is not None:
            return (lambda: oracle.ref_nbody_block(pos, vel, mass, 0, self.n)), oracle.threads(), (
                f"full {self.n}-body step, the reference's emitted OpenMP C for programs.NBODY_SHARD (extension "
                "primitives through the emitter's seams, oracle/_ref)")
        return (lambda: oracle.nbody(pos, vel, mass)), oracle.threads(), "C restatement, OpenMP"

    def parallelism(self):
        return (f"strong: 131072 bodies, 131072/{self.world} targets per rank; "
                + ("every rank's position/mass block read in place over NVLink by the force kernel "
                   "(peer pointers, all-gather fused into the fold)" if _nbody_peer() else
                   "positions/masses all-gathered (rs_allgather, NCCL) per step"))


WORKLOADS = {w.key: w for w in (Gemv, GemvOpt, Dot, DotChunked, Conv, Sgemm, SgemmNN, SgemmTiled, Nbody)}


def config_of(wl, n_gpus):
    """The `config` object: identical for both arms (the driver compares them)."""
    return {
        "workload": f"{wl.key}: BASELINE.json configs[{wl.config_index - 1}]",
        "program": wl.program,
        "sizes": wl.sizes(),
        "n_gpus": n_gpus,
        "parallelism": "1 GPU" if n_gpus == 1 else wl.parallelism(),
        "l2": ("inputs larger than L2 (>= 512 MiB of input sets used round robin)" if wl.bound == "hbm"
               else "L2 flushed between steps (256 MiB write + read, outside the events)"),
        "per_config": list(PER_CONFIG),
    }


def _nbody_peer():
    return os.environ.get("RISE_NBODY_PEER", "1") == "1"


def _dot_peer():
    return os.environ.get("RISE_DOT_PEER", "1") == "1"


def _conv_fused_halo():
    return os.environ.get("RISE_CONV_FUSED_HALO", "1") == "1"


def _time_once(fn):
    t0 = time.perf_counter()
    fn()
    return time.perf_counter() - t0


# ---------------------------------------------------------------------------
# clocks (sampled during the timed region)


class ClockSampler:
    def __init__(self, device_index: int, period_s=0.002):
        self.samples = []
        self.reasons = set()
        self.period = period_s
        self._stop = threading.Event()
        self._ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._ok = True
        except Exception:  # noqa: BLE001
            self.max_mhz = None
        self._t = threading.Thread(target=self._run, daemon=True)

    _REASONS = {
        0x0000000000000002: "applications_clocks_setting",
        0x0000000000000004: "sw_power_cap",
        0x0000000000000008: "hw_slowdown",
        0x0000000000000020: "sw_thermal_slowdown",
        0x0000000000000040: "hw_thermal_slowdown",
        0x0000000000000080: "hw_power_brake_slowdown",
    }

    def _sample(self):
        nv = self._nv
        try:
            self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
            mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            for bit, name in self._REASONS.items():
                if mask & bit:
                    self.reasons.add(name)
        except Exception:  # noqa: BLE001
            pass

    def _run(self):
        while not self._stop.is_set():
            self._sample()
            time.sleep(self.period)

    def __enter__(self):
        if self._ok:
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._ok:
            self._t.join(timeout=1)
            self._sample()  # (a short timed region still gets a sample at its end)

    def summary(self):
        med = float(np.median(self.samples)) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# our arm


class Ctx:
    """Process-wide state of our arm: rank, device, the process group."""

    def __init__(self, rank, world, local_rank):
        import torch

        self.rank, self.world, self.local_rank = rank, world, local_rank
        self.device = local_rank % max(1, torch.cuda.device_count())
        torch.cuda.set_device(self.device)
        self.dist = None
        if world > 1:
            import torch.distributed as dist

            backend = os.environ.get("RISE_DIST_BACKEND", "nccl")  # gloo: several ranks on one GPU (testing)
            if backend == "nccl" and world > torch.cuda.device_count():
                backend = "gloo"  # NCCL refuses two ranks on one device (RISE_BENCH_SHARED_GPU runs)
            if backend == "nccl":
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.device))
            else:
                dist.init_process_group(backend)
            self.dist = dist

    def barrier(self):
        if self.dist is not None:
            self.dist.barrier()

    def max_over_ranks(self, v):
        if self.dist is None:
            return v
        import torch

        t = torch.tensor([v], dtype=torch.float64, device="cuda" if self.dist.get_backend() == "nccl" else "cpu")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.dist is not None:
            self.dist.barrier()
            self.dist.destroy_process_group()


def _cubin_cache_dir():
    from paper_2201_03611_b200.runtime import cache_dir

    return cache_dir()


def measure(ctx, wl, args, steps, warmup, cpu=True):
    """One config on this rank: emit, compile, time K steps (max over ranks),
    e2e through host buffers, roofline, CPU baseline (rank 0, N = 1)."""
    import torch

    from paper_2201_03611_b200 import emit_cuda
    from paper_2201_03611_b200.run import Executable

    rank, world, dist = ctx.rank, ctx.world, ctx.dist
    compiled, nats, host = wl.local()
    t_emit = time.perf_counter()
    code = emit_cuda(compiled.unit, **wl.emit_kwargs)
    t_load = time.perf_counter()
    exe = Executable(code, nats, device=ctx.device)  # NVRTC (or the on-disk cubin cache) + module load
    t_done = time.perf_counter()
    build_times = {"emit_s": round(t_load - t_emit, 4), "nvrtc_and_load_s": round(t_done - t_load, 4),
                   "cubin_cache": "on (disk)" if _cubin_cache_dir() is not None else "off"}
    stream = torch.cuda.Stream()
    dev_in = [torch.from_numpy(np.ascontiguousarray(h).reshape(-1)).to("cuda") for h in host]
    out = torch.empty(exe.output_size, dtype=torch.float32, device="cuda")
    n_stages = len(exe.kernels)
    use_graph = n_stages > 1 and os.environ.get("RISE_BENCH_GRAPH", "1") == "1"
    keepalive = []  # peer exports of every input set stay open for the run

    def make_step(dev_in, out):
        """One step's launches on one input set (bound arguments, peer
        tables and the multi-GPU exchange included)."""
        extra = {}
        peer = None
        if exe.plan.get("peer_halo"):
            from paper_2201_03611_b200 import shard

            torch.cuda.synchronize()
            peer = shard.PeerHaloRows(dev_in[0].view(nats["n"], nats["m"]), exe.plan["stages"][0]["halo_rows"])
            dist.barrier()
            extra.update(peer.extra)
        if any(st.get("peer_exchange") for st in exe.plan["stages"]):
            from paper_2201_03611_b200 import shard

            torch.cuda.synchronize()
            peer = shard.PeerExchange()
            extra["rs_peer_table"] = peer.table
        elif exe.plan.get("peer_ranks"):
            from paper_2201_03611_b200 import shard

            torch.cuda.synchronize()
            peer = shard.PeerSources({"pos": dev_in[2], "mass": dev_in[3]}, exe.plan["stages"][0]["peer_streams"])
            dist.barrier()
            extra["rs_peer_table"] = peer.table
        keepalive.append(peer)
        launch = bound = _bound_launch(exe, dev_in, out, stream, extra)
        if use_graph:
            # a multi-kernel unit replays as one CUDA graph launch
            buffers = dict(extra)
            buffers.update({spec["name"]: value for spec, value in zip(exe.plan["inputs"], dev_in)})
            buffers[exe.plan["output"]["name"]] = out
            launch = exe.graph(buffers, stream)
        if world > 1 and not peer:
            return _distributed_step(wl, exe, dev_in, out, stream, dist, rank, world), extra, peer, None
        return launch, extra, peer, bound

    step, extra, peer, bound = make_step(dev_in, out)
    bounds = [bound]

    # L2 policy between timed steps.  HBM-bound workloads: inputs larger than
    # L2 — R input sets (>= 512 MiB = 4x L2 in total) used round robin, so every step
    # reads data evicted by the R - 1 sets read since, and the K steps run
    # back to back between two events.  The others: the L2 is flushed
    # (written, then a second buffer read) before each step, outside its events.
    set_bytes = 4 * (sum(t.numel() for t in dev_in) + out.numel())
    rotate = wl.bound == "hbm" and os.environ.get("RISE_BENCH_L2", "rotate") == "rotate"
    steps_list = [step]
    if rotate:
        n_sets = int(os.environ.get("RISE_BENCH_SETS", "0")) or max(2, -(-ROTATE_BYTES // set_bytes))
        for _ in range(n_sets - 1):
            d_in = [t.clone() for t in dev_in]
            made = make_step(d_in, torch.empty_like(out))
            steps_list.append(made[0])
            bounds.append(made[3])
        l2_text = (f"inputs larger than L2: {n_sets} input sets of {set_bytes / 2**20:.0f} MiB "
                   f"(>= 512 MiB, 4x the {L2_BYTES >> 20} MiB L2) used round robin, steps back to back")
    else:
        flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
        sweep = torch.ones(L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
        sink = torch.empty((), dtype=torch.float32, device="cuda")
        l2_text = "flushed between steps (256 MiB write + 256 MiB read sweep, outside the events)"

    def flush_l2():
        # write a buffer larger than L2, then read another one so the dirty
        # lines are written back here and not inside the next timed step
        flush.zero_()
        torch.sum(sweep, dim=0, out=sink)

    with torch.cuda.stream(stream):
        for i in range(warmup):
            if rotate:
                steps_list[i % len(steps_list)]()
            else:
                flush_l2()
                step()
    # the K back-to-back steps of the HBM-bound configs are issued the way a
    # serving loop issues them: captured once into ONE CUDA graph, one kernel
    # node per stage per step, each step on its own input set (stream-ordered:
    # a step's kernels start when the previous step's end) — one replay
    # instead of K individual launches, whose front-end gaps cost ~2 µs each
    step_graph = None
    if rotate and all(b is not None for b in bounds) and os.environ.get("RISE_BENCH_STEP_GRAPH", "1") == "1":
        from paper_2201_03611_b200 import runtime as _rt

        order = [bounds[(warmup + s_) % len(bounds)] for s_ in range(steps)]

        def record():
            for b in order:
                b()

        step_graph = _rt.Graph(record, stream)
        step_graph.upload()  # (the upload happens before the timed region, no step is executed)
    torch.cuda.synchronize()
    ctx.barrier()
    torch.cuda.synchronize()
    with ClockSampler(ctx.device) as clocks:
        if rotate:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                e0.record(stream)
                if step_graph is not None:
                    step_graph()
                else:
                    for s_ in range(steps):
                        steps_list[(warmup + s_) % len(steps_list)]()
                e1.record(stream)
        else:
            starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
            ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
            for s_ in range(steps):
                with torch.cuda.stream(stream):
                    flush_l2()
                    starts[s_].record(stream)
                    step()
                    ends[s_].record(stream)
        torch.cuda.synchronize()
        ctx.barrier()
        torch.cuda.synchronize()
    step_stats = None
    if rotate:
        total_ms = float(e0.elapsed_time(e1))
    else:
        per_step = [float(starts[s_].elapsed_time(ends[s_])) for s_ in range(steps)]
        total_ms = float(sum(per_step))
        step_stats = {"median": round(float(np.median(per_step)), 6), "best": round(min(per_step), 6),
                      "worst": round(max(per_step), 6), "note": "this rank's individually timed steps (events "
                                                                  "around each, L2 flushed before each)"}
    ms = ctx.max_over_ranks(total_ms) / steps
    total_work = wl.total_work()
    value = total_work / (ms * 1e-3) / 1e9

    # SURVEY §8 e: the replicated operand / sharded result also measured with
    # its collective inside the step (B all-gathered before the GEMM, y after
    # the GEMV)
    gathered = None
    if world > 1 and wl.key.startswith(("sgemm", "gemv")):
        try:
            gathered = _time_with_gather(ctx, wl, exe, dev_in, out, stream, steps, warmup)
        except Exception as exc:  # noqa: BLE001 - the headline line must still be printed
            gathered = {"unavailable": f"{type(exc).__name__}: {exc}"[:200]}

    # e2e: pinned host -> device, launch, device -> host, every step (each
    # rank moves its own part over its own PCIe link)
    pinned = [torch.from_numpy(np.ascontiguousarray(h).reshape(-1)).pin_memory() for h in host]
    host_out = torch.empty(exe.output_size, dtype=torch.float32).pin_memory()
    e2e_steps = max(3, min(steps, 10))
    for _ in range(2):
        exe.run_host(pinned, host_out, dev_in, out, stream, extra=extra)
    stream.synchronize()
    ctx.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        exe.run_host(pinned, host_out, dev_in, out, stream, extra=extra)
    e1.record(stream)
    stream.synchronize()
    e2e_seq_ms = e0.elapsed_time(e1) / e2e_steps
    # the same steps through the streaming API: H2D / kernels / D2H of
    # consecutive steps overlap on three streams (Executable.stream_host)
    e2e_ms = e2e_seq_ms
    if peer is None:  # (peer-memory kernels read the exported blocks, not fresh buffers)
        outs = [host_out] * e2e_steps
        exe.stream_host([pinned] * 2, [host_out] * 2, extra=extra)  # warm-up (allocations)
        ctx.barrier()
        _, pipe_ms = exe.stream_host([pinned] * e2e_steps, outs, timed=True, extra=extra)
        e2e_ms = min(pipe_ms / e2e_steps, e2e_seq_ms)
    e2e_ms = ctx.max_over_ranks(e2e_ms)
    e2e_seq_ms = ctx.max_over_ranks(e2e_seq_ms)
    # gemv with M resident in HBM (a serving system keeps its matrix on the
    # device): only x goes up and y comes down each step — reported beside e2e,
    # which moves M every step as the contract asks (SURVEY §8 e reports C2 "with
    # M pre-resident" the same way)
    resident = None
    if wl.key.startswith("gemv") and peer is None and bound is not None and world == 1:
        x_host, x_dev = pinned[1], dev_in[1]

        def one_step():
            x_dev.copy_(x_host, non_blocking=True)
            bound()
            host_out.copy_(out, non_blocking=True)

        # the step's three operations captured once into a CUDA graph (a serving
        # loop's request path): one graph launch per step instead of three
        try:
            from paper_2201_03611_b200 import runtime as _rt

            with torch.cuda.stream(stream):
                rgraph = _rt.Graph(one_step, stream)
            rgraph.upload()
            how = "one CUDA graph per step (H2D of x, the kernel, D2H of y)"
        except Exception:  # noqa: BLE001 - fall back to the three launches
            torch.cuda.synchronize()
            rgraph, how = None, "three launches per step on one stream"
        r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            for it in range(e2e_steps + 2):
                if it == 2:
                    r0.record(stream)
                rgraph() if rgraph is not None else one_step()
            r1.record(stream)
        stream.synchronize()
        r_ms = r0.elapsed_time(r1) / e2e_steps
        resident = {"value": round(total_work / (r_ms * 1e-3) / 1e9, 3), "unit": wl.metric_unit,
                    "ms_per_step": round(r_ms, 4), "h2d_bytes_per_step": 4 * x_host.numel(),
                    "d2h_bytes_per_step": 4 * host_out.numel(),
                    "path": f"M resident in HBM; every step: pinned H2D of x, the kernel, D2H of y — {how}"}
    h2d = int(sum(h.nbytes for h in host))
    d2h = int(exe.output_size * 4)

    res = None
    if rank == 0:
        peaks = _peaks()
        achieved = total_work / world / (ms * 1e-3) / 1e9  # per GPU, per step
        cpu_line = None
        if world == 1 and cpu and not args.no_cpu_baseline:
            cpu_line = cpu_baseline(wl, host)
        res = {
            "key": wl.key,
            "value": round(value, 3),
            "unit": wl.metric_unit,
            "ms_per_step": round(ms, 6),
            "steps": steps,
            "warmup": warmup,
            "scaling": "weak" if wl.scaling == "weak" and wl.key != "nbody" and world > 1 else "strong",
            "config": config_of(wl, world),
            "impl_detail": {
                "rank_sizes": {k: int(v) for k, v in nats.items()},
                "kernels": exe.kernel_names,
                "templates": exe.template_kinds,
                "l2": l2_text,
                **({"step_ms": step_stats} if step_stats is not None else {}),
                "build": dict(build_times, note="outside every timed region (the compile is cached per process "
                                                "and on disk, keyed by the kernel text)"),
                "launch": ("the K timed steps captured in one CUDA graph (one kernel node per stage per step, "
                           "each step on its own input set), replayed once" if step_graph is not None else
                           "one CUDA graph per step (Executable.graph)" if use_graph else "direct rs_launch per kernel"),
                **({"collectives": "gloo test run: host-staged"}
                   if dist is not None and dist.get_backend() != "nccl" else {}),
            },
            "e2e": {"value": round(total_work / (e2e_ms * 1e-3) / 1e9, 3), "unit": wl.metric_unit,
                    "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": d2h * world,
                    "ms_per_step": round(e2e_ms, 4),
                    "path": ("Executable.stream_host: every step's pinned H2D, kernels and D2H, consecutive steps "
                             "overlapped on three streams (double-buffered device sets)" if peer is None else
                             "Executable.run_host (peer-memory kernels read or exchange through fixed buffers: "
                             "one step at a time)") + ("" if world == 1 else "; every rank its own part over its own "
                                                                             "PCIe link"),
                    "sequential": {"value": round(total_work / (e2e_seq_ms * 1e-3) / 1e9, 3),
                                   "ms_per_step": round(e2e_seq_ms, 4),
                                   "path": "Executable.run_host: pinned H2D + launch + D2H on one stream"},
                    **({"resident_matrix": resident} if resident else {})},
            "gpu_launches": steps * n_stages,
            **({"with_collective": gathered} if gathered else {}),
            "roofline": _roofline(wl, achieved, peaks, exe),
            "cpu_baseline": cpu_line,
            "clocks": clocks.summary(),
        }
    if dist is not None:
        dist.barrier()
        for ps in keepalive:
            if ps is not None:
                ps.close()
        dist.barrier()
    del exe, dev_in, out, steps_list, step, pinned, host_out, step_graph, bounds
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return res


def cpu_baseline(wl, host):
    """The reference's CPU implementation of the same full-size config, on
    this host: best of 3 single executions for the memory-bound configs,
    one execution for the compute-bound ones (a few seconds each)."""
    fn, cores, what = wl.cpu_fn(host)
    reps = 1 if wl.compute_bound else 3
    t = min(_time_once(fn) for _ in range(reps))
    out = {"value": wl.work() / t / 1e9, "unit": wl.metric_unit, "cores": cores, "kind": _cpu_kind(what),
           "sample": f"{what}; " + ("one execution" if reps == 1 else "best of 3 executions"),
           "seconds": round(t, 4)}
    alt = wl.cpu_alt_fn(host)
    if alt is not None:
        fn, cores, what = alt
        t = min(_time_once(fn) for _ in range(reps))
        out["alt"] = {"value": wl.work() / t / 1e9, "unit": wl.metric_unit, "cores": cores,
                      "kind": _cpu_kind(what), "sample": f"{what}; best of {reps}"}
    secondary = python_reference(wl)
    if secondary is not None:
        out["secondary"] = secondary
    return out


# SURVEY.md §8 d, secondary CPU baseline: the reference's pure-Python
# functional evaluator (risec.interpreter.eval_program, interpreter.py:238;
# ~15 us per element-op on one core), at reduced sizes so it finishes in
# about a second per config (full size would take minutes to hours)
PY_REF_SIZES = {"dot": {"n": 1 << 14}, "gemv": {"n": 128, "m": 128}, "conv": {"n": 64, "m": 64},
                "sgemm_tiled": {"n": 32, "m": 32, "k": 64}, "nbody": {"n": 64}}


def python_reference(wl):
    """eval_program over the high-level program of `wl` at PY_REF_SIZES, one
    execution on one core; None when the config has no reduced size."""
    sizes = PY_REF_SIZES.get(wl.key)
    if sizes is None or os.environ.get("RISE_BENCH_PY_REF", "1") != "1":
        return None
    from paper_2201_03611_b200._ref import interpreter

    small = type(wl)()
    for k, v in sizes.items():
        setattr(small, k, v)
    compiled, nats = small.compile()
    inputs = [h.tolist() for h in small.global_inputs()]
    t0 = time.perf_counter()
    interpreter.eval_program(compiled.source_typed, nats, inputs)
    t = time.perf_counter() - t0
    shape = "x".join(str(v) for v in sizes.values())
    return {"value": round(small.work() / t / 1e9, 6), "unit": wl.metric_unit, "cores": 1, "kind": "reference",
            "sample": f"the reference's pure-Python eval_program (interpreter.py:238) on the config's RISE program at "
                      f"{shape} (reduced: SURVEY.md §8 d secondary baseline), one execution",
            "seconds": round(t, 3)}


def _cpu_kind(what):
    return "port" if "restatement" in what else "reference"


def _bound_launch(exe, dev_in, out, stream, extra=None):
    """All of a step's kernel launches with argument arrays built once
    (Executable.bind): the timed region then contains the kernels, not
    Python argument marshalling."""
    buffers = dict(extra or {})
    buffers.update({spec["name"]: value for spec, value in zip(exe.plan["inputs"], dev_in)})
    buffers[exe.plan["output"]["name"]] = out
    return exe.bind(buffers, stream)


def _time_with_gather(ctx, wl, exe, dev_in, out, stream, steps, warmup):
    """The multi-GPU step with its collective inside the timed region:
    sgemm — every rank owns 1/G of the replicated operand's rows and the
    step all-gathers it before the GEMM; gemv — the step all-gathers the
    y blocks after the GEMV.  NCCL (the process group's communicator, or the
    runtime's rs_allgather with RISE_GATHER_NATIVE=1); gloo runs (CPU test
    path) stage through host tensors."""
    import torch

    dist, rank, world = ctx.dist, ctx.rank, ctx.world
    native = dist.get_backend() == "nccl"
    if wl.key.startswith("gemv") and wl.scaling == "strong" and os.environ.get("RISE_GEMV_PEER_Y", "1") == "1":
        return _time_fused_y(ctx, wl, exe, dev_in, stream, steps, warmup)
    if wl.key.startswith("sgemm"):
        recv = dev_in[1]
        send = recv.view(world, -1)[rank].clone()
        first, what = True, "the replicated operand all-gathered from 1/G row blocks before the GEMM, every step"
    else:
        send = out
        recv = torch.empty(out.numel() * world, dtype=out.dtype, device=out.device)
        first, what = False, "the y blocks all-gathered after the GEMV, every step"
    launch = _bound_launch(exe, dev_in, out, stream)
    comm = _device_comm() if native and os.environ.get("RISE_GATHER_NATIVE", "0") == "1" else None

    def gather():
        if comm is not None:
            comm.allgather(send, recv, stream)
            return
        if native:
            with torch.cuda.stream(stream):
                dist.all_gather_into_tensor(recv, send)
            return
        with torch.cuda.stream(stream):
            parts = [torch.empty(send.numel(), dtype=send.dtype) for _ in range(world)]
            dist.all_gather(parts, send.cpu())
            recv.copy_(torch.cat(parts).to(recv.device))

    def step():
        if first:
            gather()
        launch()
        if not first:
            gather()

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    ms = ctx.max_over_ranks(e0.elapsed_time(e1) / steps)
    return {"value": round(wl.total_work() / (ms * 1e-3) / 1e9, 3), "unit": wl.metric_unit,
            "ms_per_step": round(ms, 6), "collective": what,
            "bytes_gathered_per_rank": int(recv.numel() * recv.element_size())}


def _time_fused_y(ctx, wl, exe, dev_in, stream, steps, warmup):
    """gemv with y all-gathered INSIDE the kernel: the rowfold kernel emitted
    with peer_out=N stores every row into every rank's full y (peer memory
    over NVLink) and the ranks meet once per launch in epoch-tagged slots
    (shard.PeerOutput) — one kernel per step, no collective call."""
    import torch

    from paper_2201_03611_b200 import emit_cuda, shard
    from paper_2201_03611_b200.run import Executable

    dist, world = ctx.dist, ctx.world
    compiled, nats, _host = wl.local()
    fused = Executable(emit_cuda(compiled.unit, peer_out=world), nats, device=ctx.device)
    full = torch.zeros(wl.n, dtype=torch.float32, device="cuda")
    r0, _r1 = wl.band(wl.n)
    torch.cuda.synchronize()
    po = shard.PeerOutput(full, r0)
    out = torch.empty(fused.output_size, dtype=torch.float32, device="cuda")
    launch = _bound_launch(fused, dev_in, out, stream, po.extra)
    with torch.cuda.stream(stream):
        for _ in range(warmup):
            launch()
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(steps):
            launch()
        e1.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    ms = ctx.max_over_ranks(e0.elapsed_time(e1) / steps)
    po.close()
    return {"value": round(wl.total_work() / (ms * 1e-3) / 1e9, 3), "unit": wl.metric_unit,
            "ms_per_step": round(ms, 6),
            "collective": ("y all-gathered inside the rowfold kernel: every row stored into every rank's full y over "
                           "NVLink (peer stores), epoch-tagged completion slots (emit_cuda peer_out); one kernel per "
                           "step, no collective call"),
            "bytes_gathered_per_rank": int(full.numel() * 4)}


_COMM = []


def _device_comm():
    """One NCCL communicator per process, shared by every input set's step."""
    if not _COMM:
        from paper_2201_03611_b200 import shard

        _COMM.append(shard.DeviceComm())
    return _COMM[0]


def _distributed_step(wl, exe, dev_in, out, stream, dist, rank, world):
    """The multi-GPU steps whose exchange is a separate collective (the
    fused peer-memory variants are selected in Workload.local)."""
    import torch

    bound = _bound_launch(exe, dev_in, out, stream)
    native = dist.get_backend() == "nccl"
    comm = None
    if native and wl.key in ("dot", "dot_chunked", "nbody"):
        comm = _device_comm()
    if wl.key in ("dot", "dot_chunked"):
        parts = [torch.empty(1, dtype=torch.float32, device="cuda") for _ in range(world)]
        flat = torch.empty(world, dtype=torch.float32, device="cuda")
        total = torch.empty(1, dtype=torch.float32, device="cuda")

        def step():
            bound()
            with torch.cuda.stream(stream):
                if comm is not None:
                    comm.allgather(out[:1], flat, stream)
                    gathered = list(flat.view(world, 1).unbind(0))
                else:
                    dist.all_gather(parts, out)
                    gathered = parts
                total.copy_(gathered[0])
                for p in gathered[1:]:  # rank-order fold (never an all-reduce)
                    total.add_(p)

        return step
    if wl.key == "conv":
        img, w = dev_in
        m = exe.nats["m"]
        local = img.view(-1, m)
        from paper_2201_03611_b200 import shard

        # peer-memory halo needs no collective backend (IPC works between
        # processes on one GPU too, which is how it is tested here)
        torch.cuda.synchronize()
        dist.barrier()
        halo = shard.PeerHalo(local)

        def step():  # pull the neighbours' edge rows over NVLink, then the stencil
            halo.exchange(stream)
            bound()

        step.keep = halo
        return step
    if wl.key == "nbody":
        tpos, tvel, pos, mass = dev_in
        t = exe.nats["t"]
        pos_parts = list(pos.view(world, t * 3).unbind(0))
        mass_parts = list(mass.view(world, t).unbind(0))
        mass_block = mass_parts[rank].clone()

        def step():
            with torch.cuda.stream(stream):
                if comm is not None:
                    comm.allgather(tpos, pos, stream)
                    comm.allgather(mass_block, mass, stream)
                else:
                    dist.all_gather(pos_parts, tpos)
                    dist.all_gather(mass_parts, mass_block)
            bound()

        return step
    return bound


def _roofline(wl, achieved, peaks, exe):
    extra = {}
    if wl.bound == "hbm":
        peak, unit, src = peaks["hbm_gbs"], "GB/s", peaks["source"]
        extra = {"peak_note": "the measured COPY bandwidth (reads + writes); a read-only stream (gemv, dot) "
                              "can run slightly above it (no read/write bus turnarounds)"}
    elif wl.bound == "tensor":
        # 3xTF32: three TF32 MMAs per fp32-equivalent product.  MEASURED_PEAKS
        # has no TF32 entry, so the peak is B200_PROFILING.md's dense TF32
        # (1.1 PFLOP/s) / 3; the measured bf16 burst / 2 / 3 is given beside it.
        peak, unit = TF32_DENSE_TFLOPS * 1e3 / 3.0, "GFLOP/s"
        src = "fallback (B200_PROFILING.md): dense TF32 1.1 PFLOP/s / 3 (3xTF32 fp32-equivalent)"
        bf16 = peaks.get("bf16_tflops")
        if bf16:
            alt = bf16 * 1e3 / 2 / 3.0
            extra = {"alt_peak": round(alt, 3), "alt_frac": round(achieved / alt, 4),
                     "alt_peak_source": f"MEASURED_PEAKS bf16 burst {bf16} TFLOP/s / 2 (TF32 rate) / 3"}
    else:
        peak, unit, src = FP32_SIMT_TFLOPS * 1e3, "GFLOP/s", "derived 148 SM x 128 x 2 x 1.965 GHz (FP32 SIMT)"
    traffic = None
    kern = exe.kernel_names[0] if exe.kernel_names else ""
    summary = ROOT / "profiles" / f"ncu_{wl.key}.json"
    if summary.exists():
        try:
            traffic = json.loads(summary.read_text()).get("dram_bytes_per_launch")
        except Exception:  # noqa: BLE001
            traffic = None
    return {"bound": wl.bound, "achieved": round(achieved, 3), "peak": round(peak, 3), "unit": unit,
            "frac": round(achieved / peak, 4), "traffic": traffic, "peak_source": src,
            "algorithmic_work_per_launch": wl.work() / (1 if wl.scaling == "weak" else wl.world),
            "kernel": kern, **extra}


def run_ours(args, rank, world, local_rank):
    ctx = Ctx(rank, world, local_rank)
    head_key = args.workload or HEADLINE
    keys = _per_config_keys(args)
    head = measure(ctx, WORKLOADS[head_key](rank, world, args.scaling), args, args.steps, args.warmup)
    per = {}
    for key in keys:
        if key == head_key:
            per[key] = head
            continue
        steps = args.steps if not WORKLOADS[key].compute_bound else max(3, min(args.steps, 10))
        per[key] = measure(ctx, WORKLOADS[key](rank, world, args.scaling), args, steps, args.warmup)
    ctx.close()
    if rank != 0:
        return None
    line = {
        "metric": f"{head['key']} {head['unit']} ({METRIC})",
        "value": head["value"],
        "unit": head["unit"],
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": head["ms_per_step"],
        "higher_is_better": True,
        "scaling": head["scaling"],
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (numpy default_rng seeded by config index; uniform(-1,1))",
        "config": head["config"],
        "impl_detail": head["impl_detail"],
        "e2e": head["e2e"],
        "gpu_launches": head["gpu_launches"],
        **({"with_collective": head["with_collective"]} if "with_collective" in head else {}),
        "roofline": head["roofline"],
        "cpu_baseline": head["cpu_baseline"],
        "clocks": head["clocks"],
    }
    if per:
        line["per_config"] = {k: _entry(v) for k, v in per.items()}
    return line


def _entry(r):
    keep = ("value", "unit", "ms_per_step", "steps", "warmup", "scaling", "config", "impl_detail", "e2e",
            "gpu_launches", "with_collective", "roofline", "cpu_baseline", "clocks")
    return {k: r[k] for k in keep if k in r}


def _per_config_keys(args):
    if args.configs is None:
        return list(PER_CONFIG) if args.workload is None else []
    return [k for k in args.configs.split(",") if k and k != "none"]


# ---------------------------------------------------------------------------
# reference arm: the reference's own CPU implementation


def reference_config(wl, args, world):
    """One config on the host cores: each step is ONE execution of the
    reference's emitted C/OpenMP over the full-size input."""
    host = wl.global_inputs()
    fn, cores, what = wl.cpu_fn(host)
    steps = args.steps if not wl.compute_bound else max(1, min(args.steps, 3))
    warmup = min(args.warmup, 1) if wl.compute_bound else args.warmup
    for _ in range(warmup):
        fn()
    t0 = time.perf_counter()
    for _ in range(steps):
        fn()
    elapsed = time.perf_counter() - t0
    ms = 1e3 * elapsed / steps
    value = wl.work() / (ms * 1e-3) / 1e9
    return {
        "value": round(value, 3),
        "unit": wl.metric_unit,
        "ms_per_step": round(ms, 3),
        "steps": steps,
        "warmup": warmup,
        "scaling": "strong",
        "config": config_of(wl, world),
        "cpu_baseline": {"value": round(value, 3), "unit": wl.metric_unit, "cores": cores, "kind": _cpu_kind(what),
                         "sample": f"{what}; each step one full execution", **_alt_reference(wl, host)},
        "e2e": {"value": round(value, 3), "unit": wl.metric_unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def _alt_reference(wl, host):
    alt = wl.cpu_alt_fn(host)
    if alt is None:
        return {}
    fn, cores, what = alt
    fn()
    t = min(_time_once(fn) for _ in range(3))
    return {"alt": {"value": round(wl.work() / t / 1e9, 3), "unit": wl.metric_unit, "cores": cores,
                    "kind": _cpu_kind(what), "sample": f"{what}; best of 3"}}


def run_reference(args, rank, world):
    if rank != 0:
        return None
    # every host core (torchrun sets OMP_NUM_THREADS=1 per rank; the
    # reference's OpenMP C is the only work on this host here): set before the
    # OpenMP runtime of oracle/_ref is loaded
    os.environ["OMP_NUM_THREADS"] = str(len(os.sched_getaffinity(0)))
    import oracle

    if oracle.ref_lib() is None:
        return {"impl": "reference", "unavailable": "oracle/_ref (the reference's emitted C) was not built"}
    head_key = args.workload or HEADLINE
    head = reference_config(WORKLOADS[head_key](0, world, args.scaling), args, world)
    per = {}
    for key in _per_config_keys(args):
        per[key] = head if key == head_key else reference_config(WORKLOADS[key](0, world, args.scaling), args, world)
    line = {
        "impl": "reference",
        "metric": f"{head_key} {head['unit']} ({METRIC})",
        "value": head["value"],
        "unit": head["unit"],
        "n_gpus": world,
        "steps": head["steps"],
        "warmup": head["warmup"],
        "ms_per_step": head["ms_per_step"],
        "higher_is_better": True,
        "scaling": head["scaling"],
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (numpy default_rng seeded by config index; uniform(-1,1))",
        "config": head["config"],
        "cpu_baseline": head["cpu_baseline"],
        "e2e": head["e2e"],
    }
    if per:
        line["per_config"] = {k: {kk: v for kk, v in r.items()} for k, r in per.items()}
    return line


# ---------------------------------------------------------------------------


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(n):
    """`--gpus N` without torchrun's environment: launch N ranks, one per GPU,
    through torch.distributed.run (127.0.0.1).  Fails loudly when fewer than
    N GPUs are visible (RISE_BENCH_SHARED_GPU=1 lets ranks share devices:
    the one-GPU tests)."""
    import torch

    have = torch.cuda.device_count()
    if have < n and os.environ.get("RISE_BENCH_SHARED_GPU") != "1":
        raise SystemExit(f"bench.py --gpus {n}: only {have} CUDA device(s) visible")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default=None,
                    help=f"headline config (default {HEADLINE}; giving one skips per_config unless --configs)")
    ap.add_argument("--configs", default=None, help="comma-separated per_config keys ('none' for none)")
    ap.add_argument("--scaling", choices=["strong", "weak"], default="strong")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        if args.impl == "reference":
            res = run_reference(args, 0, args.gpus)  # rank 0 alone runs (CPU)
            print(json.dumps(res), flush=True)
            return 0
        return spawn_ranks(args.gpus)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus} under a launcher with WORLD_SIZE={world}")
    if args.impl == "reference":
        res = run_reference(args, rank, world)
    else:
        res = run_ours(args, rank, world, local_rank)
    if rank == 0 and res is not None:
        print(json.dumps(res), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
