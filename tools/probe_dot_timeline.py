#!/usr/bin/env python3
"""Per-block timeline of the `reduce` (dot) kernel: the kernel text is
patched to record %globaltimer at block start, after phase 1 (the chunk
folds), and at exit (thread 0), so the launch's fixed cost can be split
into ramp (first block start -> last block start), imbalance (spread of the
phase-1 ends) and tail (last phase-1 end -> kernel end).  Probe only — not
the product kernel.

  python tools/probe_dot_timeline.py [--n 16777216] [--iters 5]
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

GT = 'asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(rs_t));'


def patched(code):
    from paper_2201_03611_b200.emit_cuda import PLAN_TAG, plan_of

    text = code.text
    plan = plan_of(text)
    st = plan["stages"][0]
    head = "unsigned long long* __restrict__ rs_partials, unsigned long long* __restrict__ rs_ticket)"
    assert head in text
    text = text.replace(head, head[:-1] + ", unsigned long long* rs_tl)")
    start = "  float rs_acc = 0.0f;\n"
    text = text.replace(start, start + f"  {{ unsigned long long rs_t; {GT} if (threadIdx.x == 0) rs_tl[3 * blockIdx.x] = rs_t; }}\n", 1)
    p2 = "  // phase 2: warp butterfly"
    text = text.replace(p2, f"  {{ unsigned long long rs_t; {GT} if (threadIdx.x == 0) rs_tl[3 * blockIdx.x + 1] = rs_t; }}\n" + p2, 1)
    p3 = "  if (!rs_last || threadIdx.x >= RS_B) return;"
    text = text.replace(p3, f"  {{ unsigned long long rs_t; {GT} if (threadIdx.x == 0) rs_tl[3 * blockIdx.x + 2] = rs_t; }}\n" + p3, 1)
    last = "      output[0] = accum;\n"
    k = text.rindex(last) + len(last)  # the reduce kernel's (the generic one comes first in the text)
    text = text[:k] + f"      {{ unsigned long long rs_t; {GT} rs_tl[3 * RS_G] = rs_t; }}\n" + text[k:]
    st["workspace"].append({"name": "rs_tl", "ctype": "int", "size": str(2 * (3 * st["grid"] + 1))})
    st["extra_args"].append({"kind": "workspace", "name": "rs_tl"})
    lines = [(PLAN_TAG + json.dumps(plan, sort_keys=True)) if ln.startswith(PLAN_TAG) else ln
             for ln in text.splitlines()]
    return "\n".join(lines) + "\n"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 24)
    ap.add_argument("--iters", type=int, default=5)
    args = ap.parse_args()
    import torch

    from paper_2201_03611_b200 import emit_cuda, programs
    from paper_2201_03611_b200.run import Executable

    code = emit_cuda(programs.compile_config("dot").unit)
    exe = Executable(patched(code), {"n": args.n})
    G = exe.plan["stages"][0]["grid"]
    sets = [[torch.rand(args.n, device="cuda") for _ in range(2)] for _ in range(4)]
    out = torch.empty(1, device="cuda")
    res = []
    for it in range(args.iters + 2):
        a, b = sets[it % 4]
        exe(a, b, out=out)
        torch.cuda.synchronize()
        tl = exe.temps()["rs_tl"].view(torch.int64)[: 3 * G + 1].cpu().numpy().astype(np.float64)
        if it < 2:
            continue
        st, p1, done, end = tl[0:3 * G:3], tl[1:3 * G:3], tl[2:3 * G:3], tl[3 * G]
        t0 = st.min()
        res.append({
            "ramp_us": (st.max() - t0) / 1e3,
            "phase1_end_min_us": (p1.min() - t0) / 1e3,
            "phase1_end_med_us": (np.median(p1) - t0) / 1e3,
            "phase1_end_max_us": (p1.max() - t0) / 1e3,
            "ticket_max_us": (done.max() - t0) / 1e3,
            "end_us": (end - t0) / 1e3,
        })
    keys = res[0].keys()
    print(json.dumps({k: round(float(np.median([r[k] for r in res])), 3) for k in keys}))


if __name__ == "__main__":
    main()
