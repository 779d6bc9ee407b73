#!/usr/bin/env python3
"""One rank's share of each strong-scaled BASELINE config, timed on ONE GPU.

This pod lends one B200 per call, so the 2/4/8-GPU runs of `bench.py --gpus
N` cannot be measured here.  What can be: the kernel each rank runs at N
ranks (rank 0's band / chunk / target block of the named shape, built by
bench.py's own Workload.local() at world N), with the single-GPU program —
the peer-memory variants are off (they wait for the other ranks), so the
exchange (peer reads, halo rows, rank-order fold of N partials) is NOT in
these numbers.  Reported: per-rank step time and the aggregate rate N ranks
would reach if the exchange were free — an upper bound that shows where
strong scaling turns launch- or tail-bound.  HBM-bound configs use input
sets >= 512 MiB round robin and K steps replayed from one CUDA graph (as
bench.py); compute-bound ones flush L2 between steps.

  python tools/probe_rank_shares.py [--steps 20] > profiles/rank_shares_r02.txt
"""
import argparse
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
os.environ["RISE_DOT_PEER"] = "0"
os.environ["RISE_CONV_FUSED_HALO"] = "0"
os.environ["RISE_NBODY_PEER"] = "0"

import numpy as np  # noqa: E402

import bench  # noqa: E402


def time_share(wl, steps, flush=False):
    import torch

    from paper_2201_03611_b200 import emit_cuda
    from paper_2201_03611_b200 import runtime as rt
    from paper_2201_03611_b200.run import Executable

    compiled, nats, host = wl.local()
    exe = Executable(emit_cuda(compiled.unit, **wl.emit_kwargs), nats)
    stream = torch.cuda.Stream()
    dev_in = [torch.from_numpy(np.ascontiguousarray(h).reshape(-1)).to("cuda") for h in host]
    out = torch.empty(exe.output_size, dtype=torch.float32, device="cuda")
    set_bytes = 4 * (sum(t.numel() for t in dev_in) + out.numel())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if wl.bound == "hbm" and not flush:
        n_sets = max(2, -(-bench.ROTATE_BYTES // set_bytes))
        sets = [(dev_in, out)] + [([t.clone() for t in dev_in], torch.empty_like(out)) for _ in range(n_sets - 1)]
        bound = [bench._bound_launch(exe, d, o, stream) for d, o in sets]
        with torch.cuda.stream(stream):
            for i in range(3):
                bound[i % n_sets]()
        graph = rt.Graph(lambda: [bound[s % n_sets]() for s in range(steps)], stream)
        graph.upload()
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            e0.record(stream)
            graph()
            e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
    else:
        step = bench._bound_launch(exe, dev_in, out, stream)
        flush = torch.empty(bench.L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
        total = 0.0
        with torch.cuda.stream(stream):
            for i in range(steps + 2):
                flush.zero_()
                e0.record(stream)
                step()
                e1.record(stream)
                torch.cuda.synchronize()
                if i >= 2:
                    total += e0.elapsed_time(e1)
        ms = total / steps
    kinds = [st["kind"] for st in exe.plan["stages"]]
    return ms, kinds, dict(nats)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--configs", default="dot,gemv,conv,sgemm_tiled,nbody")
    ap.add_argument("--rows", default="", help="instead: time the config at these row counts (n) on one rank")
    ap.add_argument("--flush", action="store_true", help="every step timed alone after an L2 flush")
    args = ap.parse_args()
    import torch

    if args.rows:
        for key in args.configs.split(","):
            cls = bench.WORKLOADS[key]
            for n in (int(v) for v in args.rows.split(",")):
                wl = type(f"{cls.__name__}N", (cls,), {"n": n})(rank=0, world=1, scaling="strong")
                ms, kinds, nats = time_share(wl, args.steps, args.flush)
                print(f"{key:12s} n={n:6d} {','.join(kinds):14s} {ms:9.4f} ms  {wl.total_work() / (ms * 1e-3) / 1e9:10.1f} "
                      f"{wl.metric_unit}", flush=True)
        return

    print(f"# {torch.cuda.get_device_name(0)}; one rank's share of each strong-scaled config (exchange excluded)")
    print("config       N  rank-0 sizes                     kernels        ms/step   aggregate if exchange free")
    for key in args.configs.split(","):
        cls = bench.WORKLOADS[key]
        base = None
        for n in (1, 2, 4, 8):
            wl = cls(rank=0, world=n, scaling="strong")
            ms, kinds, nats = time_share(wl, args.steps)
            agg = wl.total_work() / (ms * 1e-3) / 1e9
            base = base or agg
            unit = wl.metric_unit
            print(f"{key:12s} {n}  {str(nats):32s} {','.join(kinds):14s} {ms:9.4f}   {agg:10.1f} {unit} "
                  f"({agg / base:.2f}x of N=1, {agg / base / n:.2f} per GPU)", flush=True)


if __name__ == "__main__":
    main()
