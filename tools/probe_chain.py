#!/usr/bin/env python3
"""Dependent-chain latency probe (one thread): cycles per step of an
acc = acc + x chain as FADD, as FFMA with an opaque 1.0 multiplier (the
value is identical: x * 1 is exact), and as packed FADD2 — the per-element
cost of an order-preserving fold (the seqfold template)."""
import ctypes
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

SRC = r"""
#include <rise/device.cuh>
__constant__ float rs_one_c = 1.0f;
template <int MODE>
__global__ void chain(const float* x, float* out, long long* cycles, int n) {
  float acc = 0.f;
  float v[16];
  for (int i = 0; i < 16; ++i) v[i] = x[i];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (MODE == 0) acc = __fadd_rn(acc, v[k]);
      else acc = __fmaf_rn(v[k], rs_one_c, acc);
    }
  }
  long long t1 = clock64();
  out[0] = acc;
  cycles[0] = t1 - t0;
}
"""


def main():
    import torch
    from paper_2201_03611_b200 import runtime as rt

    x = torch.rand(16, device="cuda")
    out = torch.empty(1, device="cuda")
    cyc = torch.zeros(1, dtype=torch.int64, device="cuda")
    n = 1 << 16
    for mode, label in ((0, "FADD chain"), (1, "FFMA(x, 1.0 from __constant__, acc) chain")):
        mod = rt.load_module(SRC, [f"chain<{mode}>"], ["--fmad=false"])
        fn = mod.function(mod.lowered[0])
        args = [ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(cyc.data_ptr()),
                ctypes.c_int(n)]
        for _ in range(2):
            fn.launch((1, 1, 1), (1, 1, 1), args)
        torch.cuda.synchronize()
        print(f"{label}: {cyc.item() / (16 * n):.2f} cycles per step", flush=True)


if __name__ == "__main__":
    main()
