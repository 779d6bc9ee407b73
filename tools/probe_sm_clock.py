#!/usr/bin/env python3
"""The SM clock INSIDE a config's kernel (the tensor-core GEMM by default): the kernel is patched to
record clock64 and %globaltimer in thread 0 of every CTA at kernel start and
end, so each CTA's cycles / nanoseconds give the clock it actually ran at
(NVML reports the clock between samples, ncu its own replay).  Launches
follow the bench's regime (L2 flushed before each, outside the events) or
run back to back.  Probe only — not the product kernel.

  python tools/probe_gemm_sm_clock.py [--iters 30] [--mode flush|b2b]
"""
import argparse
import json
import re
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

REC = ('{{ unsigned long long c_, t_; asm volatile("mov.u64 %0, %%clock64;" : "=l"(c_)); '
       'asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); '
       'if (threadIdx.x == 0) {{ rs_ck[4 * blockIdx.x + {k}] = c_; rs_ck[4 * blockIdx.x + {k} + 1] = t_; }} }}')


def patched(code):
    from paper_2201_03611_b200.emit_cuda import PLAN_TAG, plan_of

    text = code.text
    plan = plan_of(text)
    st = plan["stages"][0]
    assert len(plan["stages"]) == 1
    m = re.search(re.escape(st["name"]) + r"\((.*?)\) \{\n(.*?)\n\}", text, re.S)
    body = m.group(2)
    text = (text[:m.end(1)] + ", unsigned long long* rs_ck) {\n  " + REC.format(k=0) + "\n" + body + "\n  "
            + REC.format(k=2) + "\n}" + text[m.end(0):])
    st.setdefault("workspace", []).append({"name": "rs_ck", "ctype": "int", "size": str(2 * 4 * 1024)})
    st["extra_args"] = st.get("extra_args", []) + [{"kind": "workspace", "name": "rs_ck"}]
    lines = [(PLAN_TAG + json.dumps(plan, sort_keys=True)) if ln.startswith(PLAN_TAG) else ln
             for ln in text.splitlines()]
    return "\n".join(lines) + "\n"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--mode", choices=["flush", "b2b"], default="flush")
    ap.add_argument("--workload", default="sgemm_tiled")
    args = ap.parse_args()
    import torch

    import bench
    from paper_2201_03611_b200 import emit_cuda
    from paper_2201_03611_b200.run import Executable

    wl = bench.WORKLOADS[args.workload]()
    compiled, nats, host = wl.local()
    exe = Executable(patched(emit_cuda(compiled.unit)), nats)
    dev = [torch.from_numpy(np.ascontiguousarray(h).reshape(-1)).to("cuda") for h in host]
    out = torch.empty(exe.output_size, device="cuda")
    flush = torch.empty(bench.L2_FLUSH_BYTES // 4, device="cuda")
    sweep = torch.ones(bench.L2_FLUSH_BYTES // 4, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(5):
        exe(*dev, out=out)
    mhz, ms = [], []
    grid = exe.kernels[0][2][0]
    for it in range(args.iters):
        if args.mode == "flush":
            flush.fill_(1.0)
            sweep.sum()
        e0.record()
        exe(*dev, out=out)
        e1.record()
        torch.cuda.synchronize()
        ck = exe.temps()["rs_ck"].view(torch.int64)[: 4 * grid].cpu().numpy().reshape(grid, 4).astype(np.float64)
        mhz.append(np.median((ck[:, 2] - ck[:, 0]) / (ck[:, 3] - ck[:, 1]) * 1e3))
        ms.append(e0.elapsed_time(e1))
    ms = np.array(ms)
    print(json.dumps({"workload": args.workload, "mode": args.mode, "ms_median": round(float(np.median(ms)), 4),
                      "ms_min": round(float(ms.min()), 4),
                      "tflops_median": round(wl.work() / (np.median(ms) * 1e-3) / 1e12, 1),
                      "in_kernel_sm_mhz": {"median": round(float(np.median(mhz)), 1), "min": round(float(min(mhz)), 1),
                                           "max": round(float(max(mhz)), 1)}}))


if __name__ == "__main__":
    main()
