#!/usr/bin/env python3
"""SM clock while the tensor-core GEMM runs back to back (no flush between
launches): NVML samples every millisecond during 200 launches of the C4
kernel, next to the achieved rate — separates the kernel's efficiency from
the power-limited clock.  Probe only.

  python tools/probe_gemm_clock.py [--iters 200]
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
    t.start()
    e0.record(stream)
    for _ in range(args.iters):
        launch()
    e1.record(stream)
    torch.cuda.synchronize()
    stop.set()
    t.join()
    ms = e0.elapsed_time(e1) / args.iters
    clk = [c for c, _p in samples]
    pw = [p for _c, p in samples]
    print(json.dumps({"workload": args.workload, "ms_per_launch": round(ms, 4),
                      "tflops": round(wl.work() / (ms * 1e-3) / 1e12, 1),
                      "sm_mhz_median": float(np.median(clk)), "sm_mhz_min": min(clk), "sm_mhz_max": max(clk),
                      "power_w_median": round(float(np.median(pw)), 1), "samples": len(samples)}))


if __name__ == "__main__":
    main()
