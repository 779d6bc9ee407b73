#!/usr/bin/env python3
"""Per-block timeline of the `stencil2d` (conv) kernel: the kernel text is
patched to record %globaltimer (thread 0 of every block) at block start, at
the top of every tile iteration, when the tile's stage is ready (mbarrier),
before the final bulk-store wait and at exit — to split a launch into ramp,
first-tile latency, per-tile time (wait vs work), and tail.  Launches run
back to back over input sets round robin (the bench's regime); the last
launch's timeline is reported.  Probe only — not the product kernel.

Measured (round 2, one B200, profiles/conv_timeline_r02.txt): at 8192² the
418 persistent blocks (19-20 tiles each) end between 72 and 95 us — blocks
on the 26 SMs that hold two blocks instead of three run faster — while a
tile's data wait is ~2.0 us and its work ~1.8 us (median).  Claiming tiles
from a counter (all of them, or only the last 1-4 rounds) measured slower
(121-127 us: the loop around a shared-memory tile index costs ~0.7 us of
work per tile at the 80-register cap), so the static walk stays.

  python tools/probe_conv_timeline.py [--n 8192] [--m 8192]
"""
import argparse
import json
import re
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

GT = 'asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(rs_tt));'
MAXIT = 40
SLOTS = 2 * MAXIT + 3


def rec(slot):
    return (f"{{ unsigned long long rs_tt; {GT} if (rs_tid == 0) "
            f"rs_tl[(size_t)blockIdx.x * {SLOTS} + ({slot})] = rs_tt; }}")


def patched(code):
    from paper_2201_03611_b200.emit_cuda import PLAN_TAG, plan_of

    text = code.text
    plan = plan_of(text)
    st = plan["stages"][0]
    assert st["kind"] == "stencil2d"
    m = re.search(r"convKernel_stencil\((.*?)\) \{", text)
    text = text[:m.end(1)] + ", unsigned long long* rs_tl" + text[m.end(1):]
    loop = re.search(r"^  for \(int rs_(t|it) = .*\{\n", text, re.M).group(0)
    text = text.replace(loop, f"  {rec(0)}\n" + loop, 1)
    top = "    const int rs_s = rs_it % RS_NSTAGE;\n"
    text = text.replace(top, top + f"    if (rs_it < {MAXIT}) {rec('1 + 2 * rs_it')}\n", 1)
    wait = "    rs_mbar_wait(&rs_bar[rs_s], (unsigned)((rs_it / RS_NSTAGE) & 1));\n"
    text = text.replace(wait, wait + f"    if (rs_it < {MAXIT}) {rec('2 + 2 * rs_it')}\n", 1)
    end = "  if (rs_tid == 0) rs_bulk_wait_all();  // the last tile's store has left shared memory\n"
    assert end in text
    text = text.replace(end, f"  {rec(2 * MAXIT + 1)}\n" + end + f"  {rec(2 * MAXIT + 2)}\n", 1)
    st.setdefault("workspace", []).append({"name": "rs_tl", "ctype": "int", "size": str(2 * 1024 * SLOTS)})
    st["extra_args"] = st.get("extra_args", []) + [{"kind": "workspace", "name": "rs_tl"}]
    lines = [(PLAN_TAG + json.dumps(plan, sort_keys=True)) if ln.startswith(PLAN_TAG) else ln
             for ln in text.splitlines()]
    return "\n".join(lines) + "\n"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--m", type=int, default=8192)
    args = ap.parse_args()
    import torch

    from paper_2201_03611_b200 import emit_cuda, programs
    from paper_2201_03611_b200.run import Executable

    n, m = args.n, args.m
    code = emit_cuda(programs.compile_config("conv").unit)
    exe = Executable(patched(code), {"n": n, "m": m})
    dyn = "schedule" in exe.plan["stages"][0]
    w = torch.tensor([[1, 2, 1], [2, 4, 2], [1, 2, 1]], dtype=torch.float32, device="cuda").reshape(-1) / 16
    n_sets = max(2, -(-(512 << 20) // (8 * n * m)))
    sets = [(torch.rand(n * m, device="cuda"), torch.empty(n * m, device="cuda")) for _ in range(n_sets)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for it in range(8):
        img, out = sets[it % n_sets]
        if it == 7:
            exe.temps()["rs_tl"].zero_()  # (the dynamic schedule's iteration counts vary per launch)
            e0.record()
        exe(img, w, out=out)
        if it == 7:
            e1.record()
    torch.cuda.synchronize()
    grid = exe.kernels[0][2][0]
    tl = exe.temps()["rs_tl"].view(torch.int64)[: grid * SLOTS].cpu().numpy().reshape(grid, SLOTS).astype(np.float64)
    start, fin0, fin = tl[:, 0], tl[:, 2 * MAXIT + 1], tl[:, 2 * MAXIT + 2]
    t0 = start.min()
    tops = tl[:, 1:2 * MAXIT + 1:2]
    ready = tl[:, 2:2 * MAXIT + 2:2]
    # (dynamic schedule: the last iteration only finds the failed claim)
    iters = [int((ready[b] > 0).sum()) - (1 if dyn else 0) for b in range(grid)]
    waits, works = [], []
    for b in range(grid):
        k = iters[b]
        for i in range(k):
            waits.append(ready[b, i] - tops[b, i])
            nxt = tops[b, i + 1] if i + 1 < k else fin0[b]
            works.append(nxt - ready[b, i])
    first_wait = ready[:, 0] - tops[:, 0]
    us = lambda v: round(float(v) / 1e3, 3)  # noqa: E731
    print(json.dumps({
        "n": n, "m": m, "grid": grid, "tiles_per_block": [min(iters), max(iters)],
        "event_us": round(e0.elapsed_time(e1) * 1e3, 2),
        "span_us": us(fin.max() - t0),
        "ramp_us": us(start.max() - t0),
        "first_tile_wait_us": {"median": us(np.median(first_wait)), "max": us(first_wait.max())},
        "tile_wait_us": {"median": us(np.median(waits)), "mean": us(np.mean(waits))},
        "tile_work_us": {"median": us(np.median(works)), "mean": us(np.mean(works))},
        "block_end_us": {"min": us(fin0.min() - t0), "median": us(np.median(fin0) - t0), "max": us(fin0.max() - t0)},
        "store_drain_us": {"median": us(np.median(fin - fin0)), "max": us((fin - fin0).max())},
    }))


if __name__ == "__main__":
    main()
