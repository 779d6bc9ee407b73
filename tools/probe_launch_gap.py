#!/usr/bin/env python3
"""Launch-issue cost vs kernel time for the dot `reduce` kernel: K launches
issued back to back (Executable.bind, one rs_launch each) against the same K
kernels replayed from one CUDA graph; CPU issue time and device time (CUDA
events) for both.  Probe only.

  python tools/probe_launch_gap.py [--k 40]
"""
import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--k", type=int, default=40)
    ap.add_argument("--workload", default="dot")
    args = ap.parse_args()
    import torch

    import bench
    from paper_2201_03611_b200 import emit_cuda, runtime
    from paper_2201_03611_b200.run import Executable

    wl = bench.WORKLOADS[args.workload]()
    compiled, nats, host = wl.local()
    exe = Executable(emit_cuda(compiled.unit), nats)
    stream = torch.cuda.Stream()
    sets = []
    for s in range(4):
        dev = [torch.from_numpy(h.reshape(-1)).to("cuda") for h in host]
        out = torch.empty(exe.output_size, device="cuda")
        bufs = {sp["name"]: d for sp, d in zip(exe.plan["inputs"], dev)}
        bufs[exe.plan["output"]["name"]] = out
        sets.append((exe.bind(bufs, stream), bufs))
    res = {}
    for _ in range(3):
        for launch, _b in sets:
            launch()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    t0 = time.perf_counter()
    for i in range(args.k):
        sets[i % 4][0]()
    t1 = time.perf_counter()
    e1.record(stream)
    torch.cuda.synchronize()
    res["direct_cpu_us_per_launch"] = (t1 - t0) * 1e6 / args.k
    res["direct_gpu_us_per_step"] = e0.elapsed_time(e1) * 1e3 / args.k

    def all_steps():
        for i in range(args.k):
            sets[i % 4][0]()

    g = runtime.Graph(all_steps, stream)
    for label, prep in (("graph_uploaded", g.upload), ("graph_replayed", g)):
        prep()
        torch.cuda.synchronize()
        e0.record(stream)
        t0 = time.perf_counter()
        g()
        t1 = time.perf_counter()
        e1.record(stream)
        torch.cuda.synchronize()
        res[f"{label}_cpu_us_total"] = (t1 - t0) * 1e6
        res[f"{label}_gpu_us_per_step"] = e0.elapsed_time(e1) * 1e3 / args.k
    print(json.dumps({k: round(v, 3) for k, v in res.items()}))


if __name__ == "__main__":
    main()
