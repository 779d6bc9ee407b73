#!/usr/bin/env python3
"""SM clock while the tensor-core GEMM runs: back to back (b2b), with the
bench's L2 flush before each launch (flush), or after 20 ms of idle (idle,
the clock recovered): NVML samples every millisecond next to the achieved
rate — separates the kernel's efficiency from the power-limited clock.
Probe only.

  python tools/probe_gemm_clock.py [--iters 200] [--mode b2b|flush|idle]
"""
import argparse
import json
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=200)
    ap.add_argument("--workload", default="sgemm_tiled")
    ap.add_argument("--mode", choices=["b2b", "flush", "idle"], default="b2b",
                    help="b2b: launches back to back; flush: the bench's L2 flush before each launch "
                         "(outside its events); idle: 20 ms of idle before each launch")
    args = ap.parse_args()
    import pynvml
    import torch

    import bench
    from paper_2201_03611_b200 import emit_cuda
    from paper_2201_03611_b200.run import Executable

    wl = bench.WORKLOADS[args.workload]()
    compiled, nats, host = wl.local()
    exe = Executable(emit_cuda(compiled.unit), nats)
    dev = [torch.from_numpy(np.ascontiguousarray(h).reshape(-1)).to("cuda") for h in host]
    out = torch.empty(exe.output_size, device="cuda")
    stream = torch.cuda.Stream()
    bufs = {sp["name"]: d for sp, d in zip(exe.plan["inputs"], dev)}
    bufs[exe.plan["output"]["name"]] = out
    launch = exe.bind(bufs, stream)
    for _ in range(5):
        launch()
    torch.cuda.synchronize()
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    samples, stop = [], threading.Event()

    def sample():
        while not stop.is_set():
            samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0))
            time.sleep(0.001)

    t = threading.Thread(target=sample, daemon=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    flush = torch.empty(bench.L2_FLUSH_BYTES // 4, device="cuda")
    sweep = torch.ones(bench.L2_FLUSH_BYTES // 4, device="cuda")
    per = []
    t.start()
    if args.mode == "b2b":
        e0.record(stream)
        for _ in range(args.iters):
            launch()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.iters
    else:
        for _ in range(args.iters):
            with torch.cuda.stream(stream):
                if args.mode == "flush":
                    flush.fill_(1.0)
                    sweep.sum()
            if args.mode == "idle":
                torch.cuda.synchronize()
                time.sleep(0.02)
            e0.record(stream)
            launch()
            e1.record(stream)
            torch.cuda.synchronize()
            per.append(e0.elapsed_time(e1))
        ms = float(np.median(per))
    stop.set()
    t.join()
    clk = [c for c, _p in samples]
    pw = [p for _c, p in samples]
    print(json.dumps({"workload": args.workload, "mode": args.mode, "ms_per_launch": round(ms, 4),
                      **({"ms_min": round(min(per), 4), "ms_max": round(max(per), 4)} if per else {}),
                      "tflops": round(wl.work() / (ms * 1e-3) / 1e12, 1),
                      "sm_mhz_median": float(np.median(clk)), "sm_mhz_min": min(clk), "sm_mhz_max": max(clk),
                      "power_w_median": round(float(np.median(pw)), 1), "samples": len(samples)}))


if __name__ == "__main__":
    main()
