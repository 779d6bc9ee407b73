#!/usr/bin/env python3
"""The strong-scaled sgemm's A row block (4096/N rows x 4096 x 4096) under
different K-split factors (tmpl_gemm.schedule patched in-process): time per
launch with the L2 flushed before each (bench regime).  Probe only.

  python tools/probe_gemm_ksplit.py [--rows 512] [--splits 1,2,4]
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=512)
    ap.add_argument("--splits", default="1,2,4")
    ap.add_argument("--iters", type=int, default=20)
    args = ap.parse_args()
    import torch

    import bench
    from paper_2201_03611_b200 import emit_cuda, programs, tmpl_gemm
    from paper_2201_03611_b200.run import Executable

    orig = tmpl_gemm.schedule
    n, m, k = args.rows, 4096, 4096
    c = programs.compile_config("sgemm_tiled")
    A = torch.rand(n * k, device="cuda") - 0.5
    B = torch.rand(k * m, device="cuda") - 0.5
    flush = torch.empty(bench.L2_FLUSH_BYTES // 4, device="cuda")
    for s in [int(v) for v in args.splits.split(",")]:
        tiles = tmpl_gemm.pair_tiles(n, m, 256)
        tmpl_gemm.schedule = (lambda M, N, K, bn, sm, persistent=True, s=s, tiles=tiles:
                              (tiles, 1) if s == 1 else (0, s))
        exe = Executable(emit_cuda(c.unit), {"n": n, "m": m, "k": k})
        out = torch.empty(n * m, device="cuda")
        stream = torch.cuda.Stream()
        bufs = {sp["name"]: d for sp, d in zip(exe.plan["inputs"], (A, B))}
        bufs[exe.plan["output"]["name"]] = out
        launch = exe.bind(bufs, stream)  # prepared launches: no host work inside the events
        ms = []
        for it in range(args.iters + 3):
            with torch.cuda.stream(stream):
                flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            launch()
            e1.record(stream)
            torch.cuda.synchronize()
            if it >= 3:
                ms.append(e0.elapsed_time(e1))
        print(json.dumps({"rows": n, "ksplit": s, "units": tiles * s, "ms_median": round(float(np.median(ms)), 4),
                          "ms_min": round(min(ms), 4)}))
    tmpl_gemm.schedule = orig


if __name__ == "__main__":
    main()
