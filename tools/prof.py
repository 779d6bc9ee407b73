#!/usr/bin/env python3
"""Launch one benchmark workload's kernels a few times on device-resident
inputs (no flush, no CPU baseline, no e2e) — the command profiled by ncu:

  ncu --set full --clock-control none -k regex:<kernel> -s <skip> -c <n> \\
      -o gpurun_out/prof_<w> python tools/prof.py --workload <w>
"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="gemv")
    ap.add_argument("--iters", type=int, default=5)
    args = ap.parse_args()
    import torch

    import bench
    from paper_2201_03611_b200 import emit_cuda
    from paper_2201_03611_b200.run import Executable

    wl = bench.WORKLOADS[args.workload]()
    compiled, nats, host = wl.local()
    exe = Executable(emit_cuda(compiled.unit, **wl.emit_kwargs), nats)
    dev = [torch.from_numpy(h.reshape(-1)).to("cuda") for h in host]
    out = torch.empty(exe.output_size, dtype=torch.float32, device="cuda")
    for _ in range(args.iters):
        exe(*dev, out=out)
    torch.cuda.synchronize()
    print("kernels:", exe.kernel_names)


if __name__ == "__main__":
    main()
