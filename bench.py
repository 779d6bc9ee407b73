#!/usr/bin/env python3
"""Benchmark of the RISE/Shine sm100a back end (the BASELINE.json metric).

One step = one execution of the hot path — the RISE program's kernel(s),
emitted by `emit_cuda` from the ImperativeUnit the reference front end
produces — over one batch of synthetic, seeded input already resident in
HBM.  Default workload: BASELINE.json configs[1], gemv fp32 8192x8192
(`mv.rise` + the toMapGlobal strategy).  Other configs: --workload.

Prints ONE JSON line (rank 0).  Timing: W warm-up steps; K timed steps
bracketed by barrier + synchronize, timed with CUDA events on the launching
stream, max over ranks.  HBM-bound workloads use inputs larger than L2: R
input sets (>= 512 MiB, 4x the L2, in total) round robin, the K steps back to back
between two events (RISE_BENCH_L2=flush selects the other mode);
compute-bound ones flush the L2 (256 MiB write + read) before every step,
outside that step's events.  `e2e` repeats the step through the
public host-buffer path (pinned H2D, launch, D2H).  `--impl reference`
times the reference's own CPU implementation (its emitted C/OpenMP,
oracle/_ref) on this host's cores instead.
"""

from __future__ import annotations

import argparse
import json
import math
import os
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


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "source": "measured (MEASURED_PEAKS.json)",
                "sm_max_mhz": d.get("sm_max_mhz", 1965.0), "bf16_tflops": d.get("bf16_tflops")}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)", "sm_max_mhz": 1965.0, "bf16_tflops": 1590.0}


# ---------------------------------------------------------------------------
# workloads: program, sizes, synthetic inputs, algorithmic work


class Workload:
    key = ""
    config_index = 0
    emit_kwargs: dict = {}

    def __init__(self, rank=0, world=1):
        self.rank, self.world = rank, world

    def inputs(self):
        raise NotImplementedError


class Gemv(Workload):
    key = "gemv"
    program = "mv.rise + toMapGlobal strategy (BASELINE.md §4 C2)"
    config_index = 2
    n = m = 8192
    metric_unit = "GB/s"
    bound = "hbm"

    def compile(self):
        from paper_2201_03611_b200 import programs

        return programs.compile_config(self.key), {"n": self.n, "m": self.m}

    def inputs(self):
        rng = np.random.default_rng(self.config_index + 1000 * self.rank)
        M = rng.uniform(-1, 1, (self.n, self.m)).astype(np.float32)
        x = rng.uniform(-1, 1, self.m).astype(np.float32)
        return [M, x]

    def work(self):  # algorithmic bytes per step (SURVEY.md §8 d)
        return 4.0 * (self.n * self.m + self.m + self.n)

    def cpu_sample(self, host):
        import oracle

        M, x = host
        rows = self.n
        t = _best_of(lambda: oracle.ref_mv(M[:rows], x), 3)
        return {"value": self.work() / t / 1e9, "unit": "GB/s", "cores": oracle.threads(), "kind": "reference",
                "sample": f"full {self.n}x{self.m} gemv, the reference's emitted OpenMP C (mv.rise + toMapGlobal, "
                          f"oracle/_ref), best of 3"}


class GemvOpt(Gemv):
    key = "gemv_opt"
    program = "mv.rise + the paper's Listing-3 strategy (mv_opt.elv), s = 32"

    def compile(self):
        from paper_2201_03611_b200 import programs

        return programs.compile_config(self.key), {"n": self.n, "m": self.m, "s": 32}


class Dot(Workload):
    key = "dot"
    program = "zip |> map(*) |> reduce(add) + fuseReduceMap;toReduceSeq (BASELINE.md §4 C1)"
    config_index = 1
    n = 1 << 24
    metric_unit = "GB/s"
    bound = "hbm"

    def compile(self):
        from paper_2201_03611_b200 import programs

        return programs.compile_config(self.key), {"n": self.n}

    def inputs(self):
        rng = np.random.default_rng(self.config_index + 1000 * self.rank)
        return [rng.uniform(-1, 1, self.n).astype(np.float32), rng.uniform(-1, 1, self.n).astype(np.float32)]

    def work(self):
        return 8.0 * self.n + 4

    def cpu_sample(self, host):
        import oracle

        a, b = host
        t = _best_of(lambda: oracle.ref_dot(a, b), 3)
        return {"value": self.work() / t / 1e9, "unit": "GB/s", "cores": 1, "kind": "reference",
                "sample": "full 2^24 dot, the reference's emitted C (sequential left fold, 1 thread), best of 3"}


class DotChunked(Dot):
    key = "dot_chunked"
    program = ("C1 (dot.rise) + the chunked-reduce strategy (gpu_rules.CHUNKED_REDUCE_STRATEGY: splitReduce(4096), "
               "...) -> split(4096) |> mapGlobal(reduceSeq) |> toMem(Global) |> reduceSeq (bit-exact)")
    emit_kwargs = {"reassociate": False}

    def compile(self):
        from paper_2201_03611_b200 import compile_program, gpu_rules, programs

        c = compile_program(programs.DOT, gpu_rules.CHUNKED_REDUCE_STRATEGY, name="dotChunked")
        return c, {"n": self.n}

    def cpu_sample(self, host):
        import oracle

        if oracle.ref_lib() is None:
            return super().cpu_sample(host)
        a, b = host
        t = _best_of(lambda: oracle.ref_dot_chunked(a, b), 3)
        return {"value": self.work() / t / 1e9, "unit": "GB/s", "cores": oracle.threads(), "kind": "reference",
                "sample": ("full 2^24 dot, the reference's emitted OpenMP C of the same chunked schedule "
                           "(chunks in parallel, then the fold of the partials), best of 3")}


class Conv(Workload):
    key = "conv"
    program = "padClamp2D + slide2D + map/reduce 3x3 (programs.CONV)"
    config_index = 3
    n = m = 8192
    metric_unit = "GB/s"
    bound = "hbm"

    def compile(self):
        from paper_2201_03611_b200 import programs

        return programs.compile_config(self.key), {"n": self.n, "m": self.m}

    def inputs(self):
        rng = np.random.default_rng(self.config_index + 1000 * self.rank)
        img = rng.uniform(-1, 1, (self.n, self.m)).astype(np.float32)
        w = (np.array([[1, 2, 1], [2, 4, 2], [1, 2, 1]], np.float32) / 16).astype(np.float32)
        return [img, w]

    def work(self):
        return 4.0 * (2 * self.n * self.m + 9)

    def cpu_sample(self, host):
        import oracle

        img, w = host
        rows = 1024
        if oracle.ref_lib() is not None:
            t = _best_of(lambda: oracle.ref_conv3x3(img[:rows], w), 3)
            kind, what = "reference", ("the reference's emitted OpenMP C for programs.CONV (extension "
                                       "primitives through the emitter's seams, oracle/_ref)")
        else:
            t = _best_of(lambda: oracle.conv3x3(img[:rows], w), 3)
            kind, what = "port", "C restatement (oracle/rise_oracle.c), OpenMP"
        return {"value": 4.0 * 2 * rows * self.m / t / 1e9, "unit": "GB/s", "cores": oracle.threads(),
                "kind": kind, "sample": f"{rows}x{self.m} band, {what}"}


class Sgemm(Workload):
    key = "sgemm"
    program = "A |> mapGlobal(arow => Bt |> mapGlobal(brow => zip |> reduceSeq)) (programs.SGEMM_BT)"
    config_index = 4
    n = m = k = 4096
    metric_unit = "GFLOP/s"
    bound = "tensor"

    def compile(self):
        from paper_2201_03611_b200 import programs

        return programs.compile_config(self.key), {"n": self.n, "m": self.m, "k": self.k}

    def inputs(self):
        rng = np.random.default_rng(self.config_index + 1000 * self.rank)
        A = rng.uniform(-1, 1, (self.n, self.k)).astype(np.float32)
        Bt = rng.uniform(-1, 1, (self.m, self.k)).astype(np.float32)
        return [A, Bt]

    def work(self):
        return 2.0 * self.n * self.m * self.k

    def cpu_sample(self, host):
        import oracle

        A, Bt = host
        rows = 64
        t = _best_of(lambda: oracle.ref_sgemm_bt(A[:rows], Bt), 2)
        return {"value": 2.0 * rows * self.m * self.k / t / 1e9, "unit": "GFLOP/s", "cores": oracle.threads(),
                "kind": "reference",
                "sample": f"{rows} rows of the 4096^3 sgemm, the reference's emitted OpenMP C (oracle/_ref)"}


class SgemmNN(Sgemm):
    key = "sgemm_nn"
    program = ("A |> mapGlobal(arow => transpose(B) |> mapGlobal(bcol => zip |> reduceSeq)) (programs.SGEMM; "
               "B row-major, MN-major tensor-core operand)")

    def compile(self):
        from paper_2201_03611_b200 import compile_program, programs

        return compile_program(programs.SGEMM, None, name="sgemm"), {"n": self.n, "m": self.m, "k": self.k}

    def inputs(self):
        A, Bt = super().inputs()
        return [A, np.ascontiguousarray(Bt.T)]

    def cpu_sample(self, host):
        A, B = host
        return super().cpu_sample([A, np.ascontiguousarray(B.T)])  # the reference C takes Bt


class Nbody(Workload):
    key = "nbody"
    program = "all-pairs map/reduce + Euler velocity step (programs.NBODY)"
    config_index = 5
    n = int(os.environ.get("RISE_NBODY_N", "131072"))  # (probes only; the config is 131072)
    metric_unit = "GFLOP/s"
    bound = "fp32-simt"

    def compile(self):
        from paper_2201_03611_b200 import programs

        return programs.compile_config(self.key), {"n": self.n}

    def inputs(self):
        rng = np.random.default_rng(self.config_index + 1000 * self.rank)
        pos = rng.uniform(-1, 1, (self.n, 3)).astype(np.float32)
        vel = np.zeros((self.n, 3), np.float32)
        mass = rng.uniform(0.5, 1.5, self.n).astype(np.float32)
        return [pos, vel, mass]

    def work(self):
        return 20.0 * self.n * self.n

    def cpu_sample(self, host):
        import oracle

        pos, vel, mass = host
        count = 256
        if oracle.ref_lib() is not None:
            t = _best_of(lambda: oracle.ref_nbody_block(pos, vel, mass, 0, count), 2)
            kind, what = "reference", ("the reference's emitted OpenMP C for programs.NBODY_SHARD (extension "
                                       "primitives through the emitter's seams, oracle/_ref)")
        else:
            t = _best_of(lambda: oracle.nbody(pos, vel, mass, 0, count), 2)
            kind, what = "port", "C restatement, OpenMP"
        return {"value": 20.0 * count * self.n / t / 1e9, "unit": "GFLOP/s", "cores": oracle.threads(),
                "kind": kind, "sample": f"{count} target bodies x {self.n} sources, {what}"}


WORKLOADS = {w.key: w for w in (Gemv, GemvOpt, Dot, DotChunked, Conv, Sgemm, SgemmNN, Nbody)}


def _best_of(fn, k):
    best = math.inf
    for _ in range(k):
        t0 = time.perf_counter()
        fn()
        best = min(best, time.perf_counter() - t0)
    return best


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

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self._REASONS.items():
                    if mask & bit:
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self._ok:
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._ok:
            self._t.join(timeout=1)

    def summary(self):
        med = float(np.median(self.samples)) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# our arm


def run_ours(args, rank, world, local_rank):
    import torch

    from paper_2201_03611_b200 import emit_cuda
    from paper_2201_03611_b200.run import Executable

    device = local_rank % max(1, torch.cuda.device_count())
    torch.cuda.set_device(device)
    dist = None
    if world > 1:
        import torch.distributed as dist

        backend = os.environ.get("RISE_DIST_BACKEND", "nccl")  # gloo: several ranks on one GPU (testing)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", device))
        else:
            dist.init_process_group(backend)
    wl = WORKLOADS[args.workload](rank, world)
    compiled, nats = wl.compile()
    host = wl.inputs()
    if world > 1:
        compiled, nats, host = _distributed_variant(wl, compiled, nats, host, rank, world)
    code = emit_cuda(compiled.unit, **wl.emit_kwargs)
    exe = Executable(code, nats, device=device)
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
        peer_sources = None
        if exe.plan.get("peer_halo"):
            from paper_2201_03611_b200 import shard

            torch.cuda.synchronize()
            peer_sources = shard.PeerHaloRows(dev_in[0].view(nats["n"], nats["m"]), exe.plan["stages"][0]["halo_rows"])
            dist.barrier()
            extra.update(peer_sources.extra)
        if any(st.get("peer_exchange") for st in exe.plan["stages"]):
            from paper_2201_03611_b200 import shard

            torch.cuda.synchronize()
            peer_sources = shard.PeerExchange()
            extra["rs_peer_table"] = peer_sources.table
        elif exe.plan.get("peer_ranks"):
            from paper_2201_03611_b200 import shard

            torch.cuda.synchronize()
            peer_sources = shard.PeerSources({"pos": dev_in[2], "mass": dev_in[3]},
                                             exe.plan["stages"][0]["peer_streams"])
            dist.barrier()
            extra["rs_peer_table"] = peer_sources.table
        keepalive.append(peer_sources)
        launch = _bound_launch(exe, dev_in, out, stream, extra)
        if use_graph:
            # a multi-kernel unit replays as one CUDA graph launch
            buffers = dict(extra)
            buffers.update({spec["name"]: value for spec, value in zip(exe.plan["inputs"], dev_in)})
            buffers[exe.plan["output"]["name"]] = out
            launch = exe.graph(buffers, stream)
        if world > 1 and not peer_sources:
            return _distributed_step(wl, exe, dev_in, out, stream, dist, rank, world), extra, peer_sources
        return launch, extra, peer_sources

    step, extra, peer_sources = make_step(dev_in, out)

    # L2 policy between timed steps.  HBM-bound workloads: inputs larger than
    # L2 — R input sets (>= 512 MiB = 4x L2 in total) used round robin, so every step
    # reads data evicted by the R - 1 sets read since, and the K steps run
    # back to back between two events.  The others: the L2 is flushed
    # (written, then a second buffer read) before each step, outside its events.
    set_bytes = 4 * (sum(t.numel() for t in dev_in) + out.numel())
    rotate = wl.bound == "hbm" and os.environ.get("RISE_BENCH_L2", "rotate") == "rotate"
    if rotate:
        n_sets = int(os.environ.get("RISE_BENCH_SETS", "0")) or max(2, -(-ROTATE_BYTES // set_bytes))
        steps = [step]
        for _ in range(n_sets - 1):
            d_in = [t.clone() for t in dev_in]
            steps.append(make_step(d_in, torch.empty_like(out))[0])
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
        for i in range(args.warmup):
            if rotate:
                steps[i % len(steps)]()
            else:
                flush_l2()
                step()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clocks:
        if rotate:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                e0.record(stream)
                for s_ in range(args.steps):
                    steps[(args.warmup + s_) % len(steps)]()
                e1.record(stream)
        else:
            starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
            ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
            for s_ in range(args.steps):
                with torch.cuda.stream(stream):
                    flush_l2()
                    starts[s_].record(stream)
                    step()
                    ends[s_].record(stream)
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
    if rotate:
        total_ms = float(e0.elapsed_time(e1))
    else:
        total_ms = float(sum(starts[s_].elapsed_time(ends[s_]) for s_ in range(args.steps)))
    if dist is not None:
        t = torch.tensor([total_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms = total_ms / args.steps
    strong = world > 1 and wl.key == "nbody"
    total_work = wl.work() if strong else wl.work() * world
    value = total_work / (ms * 1e-3) / 1e9

    # SURVEY §8 e: the replicated operand / sharded result also measured with
    # its collective inside the step (B all-gathered before the GEMM, y after
    # the GEMV)
    gathered = None
    if world > 1 and wl.key in ("sgemm", "sgemm_nn", "gemv", "gemv_opt"):
        try:
            gathered = _time_with_gather(wl, exe, dev_in, out, stream, dist, rank, world, args)
        except Exception as exc:  # noqa: BLE001 - the headline line must still be printed
            gathered = {"unavailable": f"{type(exc).__name__}: {exc}"[:200]}

    # e2e: pinned host -> device, launch, device -> host, every step
    pinned = [torch.from_numpy(h.reshape(-1)).pin_memory() for h in host]
    host_out = torch.empty(exe.output_size, dtype=torch.float32).pin_memory()
    e2e_steps = max(3, min(args.steps, 10))
    for _ in range(2):
        exe.run_host(pinned, host_out, dev_in, out, stream, extra=extra)
    stream.synchronize()
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
    if peer_sources is None:  # (peer-source kernels read the exported blocks, not fresh buffers)
        outs = [host_out] * e2e_steps
        exe.stream_host([pinned] * 2, [host_out] * 2, extra=extra)  # warm-up (allocations)
        _, pipe_ms = exe.stream_host([pinned] * e2e_steps, outs, timed=True, extra=extra)
        e2e_ms = min(pipe_ms / e2e_steps, e2e_seq_ms)
    if dist is not None:
        t = torch.tensor([e2e_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    h2d = int(sum(h.nbytes for h in host))
    d2h = int(exe.output_size * 4)

    result = None
    if rank == 0:
        peaks = _peaks()
        achieved = total_work / world / (ms * 1e-3) / 1e9  # per GPU, per step
        roof = _roofline(wl, achieved, peaks, args)
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = wl.cpu_sample(host)
        result = {
            "metric": f"{wl.key} {wl.metric_unit} (per-benchmark GFLOP/s or GB/s vs B200 roofline)",
            "value": round(value, 3),
            "unit": wl.metric_unit,
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms, 6),
            "higher_is_better": True,
            "scaling": "strong" if strong else "weak",
            "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic (numpy default_rng seeded by config index; uniform(-1,1))",
            "config": {
                "workload": f"{wl.key}: BASELINE.json configs[{wl.config_index - 1}]",
                "program": wl.program,
                "sizes": nats,
                "kernels": exe.kernel_names,
                "templates": exe.template_kinds,
                "l2": l2_text,
                "launch": ("one CUDA graph per step (Executable.graph)" if n_stages > 1
                           and os.environ.get("RISE_BENCH_GRAPH", "1") == "1" else "direct rs_launch per kernel"),
                "parallelism": _parallelism_text(wl, world) + (
                    "" if dist is None or dist.get_backend() == "nccl"
                    else " [gloo test run: collectives host-staged]"),
            },
            "e2e": {"value": round(total_work / (e2e_ms * 1e-3) / 1e9, 3), "unit": wl.metric_unit,
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": round(e2e_ms, 4),
                    "path": ("Executable.stream_host: every step's pinned H2D, kernels and D2H, consecutive steps "
                             "overlapped on three streams (double-buffered device sets)" if peer_sources is None else
                             "Executable.run_host (peer-memory kernels read or exchange through fixed buffers: "
                             "one step at a time)"),
                    "sequential": {"value": round(total_work / (e2e_seq_ms * 1e-3) / 1e9, 3),
                                   "ms_per_step": round(e2e_seq_ms, 4),
                                   "path": "Executable.run_host: pinned H2D + launch + D2H on one stream"}},
            "gpu_launches": args.steps * n_stages,
            **({"with_collective": gathered} if gathered else {}),
            "roofline": roof,
            "cpu_baseline": cpu,
            "clocks": clocks.summary(),
        }
    if dist is not None:
        dist.barrier()
        for ps in keepalive:
            if ps is not None:
                ps.close()
        dist.barrier()
        dist.destroy_process_group()
    return result


def _parallelism_text(wl, world):
    if world == 1:
        return "1 GPU"
    return {
        "gemv": f"weak: rank r owns an 8192-row band of an ({world}x8192) x 8192 matrix, x replicated, y sharded",
        "gemv_opt": f"weak: rank r owns an 8192-row band of an ({world}x8192) x 8192 matrix, x replicated",
        "sgemm": f"weak: rank r owns a 4096-row block of A ({world}x4096 rows), B replicated",
        "sgemm_nn": f"weak: rank r owns a 4096-row block of A ({world}x4096 rows), B replicated",
        "dot": ("weak: rank r owns a 2^24 chunk; " + (
            "the reduce kernel publishes its total into every rank's slots over NVLink (peer memory) and folds "
            "the totals in rank order (exchange fused into the kernel)" if _dot_peer() else
            "partials all-gathered (rs_allgather, NCCL) and folded in rank order")),
        "dot_chunked": "weak: rank r owns a 2^24 chunk; partials all-gathered (rs_allgather, NCCL), rank-order fold",
        "conv": ("weak: rank r owns an 8192-row band; " + (
            "the stencil kernel reads the neighbours' edge rows in place over NVLink (peer pointers, "
            "halo exchange fused into the border-tile staging)" if _conv_fused_halo() else
            "halo rows pulled from the neighbours' bands over NVLink (rs_halo_exchange, CUDA IPC) per step")),
        "nbody": (f"strong: 131072 bodies, {131072 // world} targets per rank; "
                  + ("every rank's position/mass block read in place over NVLink by the force kernel "
                     "(peer pointers, all-gather fused into the fold)" if _nbody_peer() else
                     "positions/masses all-gathered (rs_allgather, NCCL) per step")),
    }[wl.key]


def _distributed_variant(wl, compiled, nats, host, rank, world):
    """Per-rank program, sizes and inputs of the multi-GPU decomposition
    (paper_2201_03611_b200/shard.py)."""
    from paper_2201_03611_b200 import compile_program, programs

    if wl.key == "dot" and _dot_peer():
        # the fused variant: each rank's reduce kernel publishes its total into
        # every rank's exchange slots (peer memory) and folds them in rank order
        wl.emit_kwargs = {"peer_ranks": world}
        return compiled, nats, host
    if wl.key == "conv" and _conv_fused_halo():
        # the fused variant: the stencil kernel reads its neighbours' edge rows
        # in place (peer pointers), so the band is exactly this rank's rows
        wl.emit_kwargs = {"peer_halo": True}
        return compiled, nats, host
    if wl.key == "conv":
        img, w = host
        local = np.empty((img.shape[0] + 2, img.shape[1]), np.float32)
        local[1:-1] = img
        local[0], local[-1] = img[0], img[-1]
        nats = {"n": img.shape[0] + 2, "m": img.shape[1]}
        return compiled, nats, [local, w]
    if wl.key == "nbody":
        n = wl.n
        if n % world:
            raise SystemExit(f"nbody: {n} bodies do not split over {world} ranks")
        t = n // world
        rng = np.random.default_rng(wl.config_index)  # the same global system on every rank
        pos = rng.uniform(-1, 1, (n, 3)).astype(np.float32)
        mass = rng.uniform(0.5, 1.5, n).astype(np.float32)
        t0 = rank * t
        c = compile_program(programs.NBODY_SHARD, None, name="nbodyShard")
        if _nbody_peer():
            # the fused variant: each rank holds only its block; the kernel
            # reads every other block in place over NVLink (peer pointers)
            wl.emit_kwargs = {"peer_ranks": world}
            blk = pos[t0:t0 + t]
            return c, {"t": t, "n": n}, [blk, np.zeros((t, 3), np.float32), blk, mass[t0:t0 + t]]
        return c, {"t": t, "n": n}, [pos[t0:t0 + t], np.zeros((t, 3), np.float32), pos, mass]
    return compiled, nats, host


def _nbody_peer():
    return os.environ.get("RISE_NBODY_PEER", "1") == "1"


def _dot_peer():
    return os.environ.get("RISE_DOT_PEER", "1") == "1"


def _conv_fused_halo():
    return os.environ.get("RISE_CONV_FUSED_HALO", "1") == "1"


def _bound_launch(exe, dev_in, out, stream, extra=None):
    """All of a step's kernel launches with argument arrays built once
    (Executable.bind): the timed region then contains the kernels, not
    Python argument marshalling."""
    buffers = dict(extra or {})
    buffers.update({spec["name"]: value for spec, value in zip(exe.plan["inputs"], dev_in)})
    buffers[exe.plan["output"]["name"]] = out
    return exe.bind(buffers, stream)


def _time_with_gather(wl, exe, dev_in, out, stream, dist, rank, world, args):
    """The multi-GPU step with its collective inside the timed region:
    sgemm — every rank owns 1/G of the replicated operand's rows and the
    step all-gathers it before the GEMM; gemv — the step all-gathers the
    y blocks after the GEMV.  NCCL (the process group's communicator, or the
    runtime's rs_allgather with RISE_GATHER_NATIVE=1); gloo runs (CPU test
    path) stage through host tensors."""
    import torch

    native = dist.get_backend() == "nccl"
    if wl.key.startswith("sgemm"):
        recv = dev_in[1]
        send = recv.view(world, -1)[rank].clone()
        first, what = True, "the replicated operand all-gathered from 1/G row blocks before the GEMM, every step"
    else:
        send = out
        recv = torch.empty(out.numel() * world, dtype=out.dtype, device=out.device)
        first, what = False, "the y blocks all-gathered after the GEMV, every step"
    launch = _bound_launch(exe, dev_in, out, stream)
    # the process group's own NCCL communicator (no second communicator for a
    # reporting variant; RISE_GATHER_NATIVE=1 uses the runtime's rs_allgather)
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

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    t = torch.tensor([e0.elapsed_time(e1) / args.steps], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    return {"value": round(wl.work() * world / (ms * 1e-3) / 1e9, 3), "unit": wl.metric_unit,
            "ms_per_step": round(ms, 6), "collective": what,
            "bytes_gathered_per_rank": int(recv.numel() * recv.element_size())}


_COMM = []


def _device_comm():
    """One NCCL communicator per process, shared by every input set's step."""
    if not _COMM:
        from paper_2201_03611_b200 import shard

        _COMM.append(shard.DeviceComm())
    return _COMM[0]


def _distributed_step(wl, exe, dev_in, out, stream, dist, rank, world):
    import torch

    bound = _bound_launch(exe, dev_in, out, stream)

    class _Exe:  # the distributed steps call exe(...) -> the bound launch
        nats = exe.nats

        def __call__(self, *a, **k):
            bound()

    exe = _Exe()
    # NCCL runs: the data path goes through the native runtime's collectives
    # (rs_allgather over NCCL, rs_halo_exchange over peer memory); gloo runs
    # (CPU test path, several ranks per GPU) move host-staged tensors
    native = dist.get_backend() == "nccl"
    comm = None
    if native and wl.key in ("dot", "dot_chunked", "nbody"):
        comm = _device_comm()
    if wl.key in ("dot", "dot_chunked"):
        parts = [torch.empty(1, dtype=torch.float32, device="cuda") for _ in range(world)]
        flat = torch.empty(world, dtype=torch.float32, device="cuda")
        total = torch.empty(1, dtype=torch.float32, device="cuda")

        def step():
            exe(*dev_in, out=out, stream=stream)
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

        host_staged = not native  # gloo P2P moves CPU tensors only (test path)
        stage = torch.empty((4, m), dtype=torch.float32) if host_staged else None
        if native or os.environ.get("RISE_PEER_HALO", "1") == "1":
            # peer-memory halo needs no collective backend (IPC works between
            # processes on one GPU too, which is how it is tested here)
            from paper_2201_03611_b200 import shard

            torch.cuda.synchronize()
            dist.barrier()
            halo = shard.PeerHalo(local)

            def step():  # pull the neighbours' edge rows over NVLink, then the stencil
                halo.exchange(stream)
                exe(*dev_in, out=out, stream=stream)

            return step

        def step():
            with torch.cuda.stream(stream):
                if host_staged:
                    stage[0].copy_(local[1])
                    stage[1].copy_(local[-2])
                    send_top, send_bot, recv_top, recv_bot = stage[0], stage[1], stage[2], stage[3]
                else:
                    send_top, send_bot, recv_top, recv_bot = local[1], local[-2], local[0], local[-1]
                ops = []
                if rank > 0:
                    ops += [dist.P2POp(dist.isend, send_top, rank - 1), dist.P2POp(dist.irecv, recv_top, rank - 1)]
                if rank < world - 1:
                    ops += [dist.P2POp(dist.isend, send_bot, rank + 1), dist.P2POp(dist.irecv, recv_bot, rank + 1)]
                for req in dist.batch_isend_irecv(ops):
                    req.wait()
                if host_staged:
                    if rank > 0:
                        local[0].copy_(recv_top)
                    if rank < world - 1:
                        local[-1].copy_(recv_bot)
            exe(*dev_in, out=out, stream=stream)

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
            exe(*dev_in, out=out, stream=stream)

        return step

    def step():
        exe(*dev_in, out=out, stream=stream)

    return step


def _roofline(wl, achieved, peaks, args):
    if wl.bound == "hbm":
        peak, unit, src = peaks["hbm_gbs"], "GB/s", peaks["source"]
    elif wl.bound == "tensor":
        # the TF32 MMA rate is half the BF16 rate on sm_100; cuBLAS's own TF32
        # sgemm reaches less than that, so the larger of the two is the roof
        cublas = _tf32_peak()
        bf16 = peaks.get("bf16_tflops")
        if bf16 and bf16 * 1e3 / 2 > cublas:
            peak, src = bf16 * 1e3 / 2 / 3.0, (f"MEASURED_PEAKS bf16 {bf16} TFLOP/s / 2 (TF32 MMA rate) / 3 "
                                               f"(3xTF32 fp32-equivalent); cuBLAS TF32 sgemm measured "
                                               f"{cublas / 1e3:.1f} TFLOP/s")
        else:
            peak, src = cublas / 3.0, "measured cuBLAS TF32 / 3 (3xTF32 fp32-equivalent)"
        unit = "GFLOP/s"
    else:
        peak, unit, src = FP32_SIMT_TFLOPS * 1e3, "GFLOP/s", "derived 148 SM x 128 x 2 x 1.965 GHz"
    traffic = None
    summary = ROOT / "profiles" / f"ncu_{wl.key}.json"
    if summary.exists():
        try:
            traffic = json.loads(summary.read_text()).get("dram_bytes_per_launch")
        except Exception:  # noqa: BLE001
            traffic = None
    out = {"bound": wl.bound, "achieved": round(achieved, 3), "peak": round(peak, 3), "unit": unit,
           "frac": round(achieved / peak, 4), "traffic": traffic, "peak_source": src,
           "algorithmic_work_per_launch": wl.work()}
    if wl.bound == "tensor":
        # context: B200_PROFILING.md's nominal dense TF32 (1.1 PFLOP/s) / 3
        out["nominal_peak"] = round(1100e3 / 3.0, 3)
        out["frac_of_nominal"] = round(achieved / (1100e3 / 3.0), 4)
    return out


def _tf32_peak():
    import torch

    torch.backends.cuda.matmul.allow_tf32 = True
    a = torch.randn(8192, 8192, device="cuda")
    b = torch.randn(8192, 8192, device="cuda")
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    best = math.inf
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    torch.backends.cuda.matmul.allow_tf32 = False
    return 2 * 8192 ** 3 / (best * 1e-3) / 1e9


# ---------------------------------------------------------------------------
# reference arm: the reference's own CPU implementation


def run_reference(args, rank, world):
    if rank != 0:
        return None
    import oracle

    wl = WORKLOADS[args.workload](0, 1)
    host = wl.inputs()
    if oracle.ref_lib() is None and wl.key in ("gemv", "gemv_opt", "dot", "sgemm"):
        return {"impl": "reference", "unavailable": "oracle/_ref (the reference's emitted C) was not built"}
    for _ in range(args.warmup):
        wl.cpu_sample(host)
    t0 = time.perf_counter()
    vals = []
    sample = None
    for _ in range(args.steps):
        sample = wl.cpu_sample(host)
        vals.append(sample["value"])
    elapsed = time.perf_counter() - t0
    value = float(np.median(vals))
    return {
        "impl": "reference",
        "metric": f"{wl.key} {wl.metric_unit} (per-benchmark GFLOP/s or GB/s vs B200 roofline)",
        "value": round(value, 3),
        "unit": sample["unit"],
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(1e3 * elapsed / args.steps, 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (numpy default_rng seeded by config index; uniform(-1,1))",
        "config": {"workload": f"{wl.key}: BASELINE.json configs[{wl.config_index - 1}]", "program": wl.program},
        "cpu_baseline": {"value": round(value, 3), "unit": sample["unit"], "cores": sample["cores"],
                         "kind": sample["kind"], "sample": sample["sample"]},
        "e2e": {"value": round(value, 3), "unit": sample["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="gemv")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(1)))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        res = run_reference(args, rank, world)
    else:
        res = run_ours(args, rank, world, local_rank)
    if rank == 0 and res is not None:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
