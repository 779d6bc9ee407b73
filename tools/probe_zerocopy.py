#!/usr/bin/env python3
"""Host -> GPU bandwidth: the copy engine (cudaMemcpyAsync from pinned memory)
against SM loads straight from pinned host memory (zero-copy, UVA pointer),
for the e2e figure's PCIe leg.  Probe only."""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2201_03611_b200 import runtime  # noqa: E402

SRC = r'''
extern "C" __global__ void zsum(const float4* __restrict__ p, long long n4, float* out) {
  float acc = 0.f;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    float4 v = __ldcs(p + i);
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 1234.5f) out[0] = acc;
}
'''
n = 268435456 // 4
h = torch.empty(n, dtype=torch.float32).pin_memory()
h.uniform_()
d = torch.empty(n, dtype=torch.float32, device="cuda")
out = torch.zeros(1, device="cuda")
cubin, names = runtime.compile_cubin(SRC, ["zsum"])
fn = runtime.Module(cubin, names).function(names[0] or "zsum")


def t(f, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


print("copy engine H2D", round(268.4 / t(lambda: d.copy_(h, non_blocking=True)), 1), "GB/s")
for blocks, threads in ((148, 1024), (296, 1024), (592, 512), (1184, 256), (2368, 256)):
    args = [ctypes.c_void_p(h.data_ptr()), ctypes.c_longlong(n // 4), ctypes.c_void_p(out.data_ptr())]
    ms = t(lambda: fn.launch((blocks, 1, 1), (threads, 1, 1), args))
    print(f"zero-copy SM loads {blocks}x{threads}", round(268.4 / ms, 1), "GB/s")
