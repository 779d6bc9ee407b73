#!/usr/bin/env python3
"""Per-pair timeline of the persistent tcgen05 GEMM: the kernel is compiled
with RS_GEMM_TIMELINE_OFFSET so CTA rank 0 of every pair records
%globaltimer at 0 the MMA issuer's start of unit i, 1 after it got a free
TMEM slot, 2 at its first ready stage, 3 after its last commit, 4 when the
epilogue sees the accumulator, 6 after a split tile's parts arrived, 5 at
the epilogue's end.  Prints the medians / maxima of each phase and the
last unit's end per pair.  Probe only.

  python tools/probe_gemm_timeline.py [--rows 4096] [--mode flush]
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
    ap.add_argument("--rows", type=int, default=4096)
    ap.add_argument("--iters", type=int, default=5)
    args = ap.parse_args()
    import torch

    import bench
    from paper_2201_03611_b200 import emit_cuda, programs
    from paper_2201_03611_b200.emit_cuda import PLAN_TAG, plan_of
    from paper_2201_03611_b200.run import Executable

    n, m, k = args.rows, 4096, 4096
    code = emit_cuda(programs.compile_config("sgemm_tiled").unit)
    text = code.text
    plan = plan_of(text)
    st = plan["stages"][0]
    ws = next(w for w in st["workspace"] if w["ctype"] == "float")
    off = 74 * 256 * 256  # floats past the normal workspace (even: 8-byte aligned)
    ws["size"] = f"({ws['size']}) + {off} + 74 * 16 * 8 * 2"
    text = "\n".join((PLAN_TAG + json.dumps(plan, sort_keys=True)) if ln.startswith(PLAN_TAG) else ln
                     for ln in text.splitlines()) + "\n"
    text = text.replace("#include <rise/gemm_tc.cuh>", f"#define RS_GEMM_TIMELINE_OFFSET ({off}LL)\n#include <rise/gemm_tc.cuh>")
    exe = Executable(text, {"n": n, "m": m, "k": k})
    A = torch.rand(n * k, device="cuda") - 0.5
    B = torch.rand(k * m, device="cuda") - 0.5
    out = torch.empty(n * m, device="cuda")
    stream = torch.cuda.Stream()
    bufs = {sp["name"]: d for sp, d in zip(exe.plan["inputs"], (A, B))}
    bufs[exe.plan["output"]["name"]] = out
    launch = exe.bind(bufs, stream)
    flush = torch.empty(bench.L2_FLUSH_BYTES // 4, device="cuda")
    for _ in range(args.iters):
        with torch.cuda.stream(stream):
            flush.zero_()
            tl_buf = exe.temps()[ws["name"]]
            tl_buf[off:].zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        launch()
        e1.record(stream)
        torch.cuda.synchronize()
    tl = exe.temps()[ws["name"]][off:off + 74 * 16 * 8 * 2].view(torch.int64).cpu().numpy()
    tl = tl.reshape(74, 16, 8).astype(np.float64)
    t0 = tl[:, 0, 0][tl[:, 0, 0] > 0].min()
    ph = {"wait_tmem_slot": (1, 0), "wait_first_stage": (2, 1), "mma_issue": (3, 2), "mma_drain_to_epilogue": (4, 3),
          "parts_wait": (6, 4), "epilogue_after_parts": (5, 6)}
    res = {"rows": n, "event_ms": round(e0.elapsed_time(e1), 4)}
    units = (tl[:, :, 0] > 0).sum(axis=1)
    res["units_per_pair"] = [int(units.min()), int(units.max())]
    for name, (a, b) in ph.items():
        v = []
        for p in range(74):
            for i in range(units[p]):
                if tl[p, i, a] > 0 and tl[p, i, b] > 0:
                    v.append((tl[p, i, a] - tl[p, i, b]) / 1e3)
        if v:
            res[name + "_us"] = {"median": round(float(np.median(v)), 2), "max": round(float(np.max(v)), 2),
                                 "sum_median_per_pair": None}
    ends = [(tl[p, units[p] - 1, 5] - t0) / 1e3 for p in range(74) if units[p] > 0]
    res["pair_end_us"] = {"min": round(min(ends), 1), "median": round(float(np.median(ends)), 1), "max": round(max(ends), 1)}
    first = [(tl[p, 0, 2] - t0) / 1e3 for p in range(74) if units[p] > 0]
    res["first_stage_ready_us"] = {"median": round(float(np.median(first)), 2), "max": round(max(first), 2)}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
