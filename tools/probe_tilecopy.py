#!/usr/bin/env python3
"""Tile-shape probe for the stencil's data movement: a persistent kernel that
moves an 8192^2 fp32 image exactly as the stencil2d template does — per
tile one (or two) 2-D TMA loads of the (TR + 2) x (TC + 8) footprint into a
ring stage, a register window, the interior written back to shared memory
as a [TR][TC] tile and one TMA tile store — with no arithmetic.  Timed over
two input sets round robin, steps back to back (the bench's regime), for
several tile shapes: what the movement alone reaches, per shape."""
import ctypes
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

SRC = r"""
#include <rise/device.cuh>
template <int H, int W, int TR, int TC, int NB, int NSTAGE, int PAD, int MODE>
__global__ void __launch_bounds__(256) tilecopy(float* out, const __grid_constant__ rs_tmap map,
                                                const __grid_constant__ rs_tmap omap) {
  constexpr int SR = TR + 2, SW = TC + 2 * PAD, BW = SW / NB;  // MODE 0 copy, 1 loads only, 2 stores only
  constexpr int BS = (SR * BW + 31) / 32 * 32;  // box regions stay 128-byte aligned
  constexpr int STAGE = NB * BS;
  constexpr int NTX = W / TC, NTILES = NTX * (H / TR);
  extern __shared__ __align__(128) unsigned char dsm[];
  float* buf = reinterpret_cast<float*>(dsm + ((128u - (rs_smem_addr(dsm) & 127u)) & 127u));
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(buf + NSTAGE * STAGE);
  const int tid = threadIdx.x;
  auto issue = [&](int t, int s) {
    const int r0 = (t / NTX) * TR, c0 = (t % NTX) * TC;
    rs_fence_proxy_async();
    if (MODE == 2) { rs_mbar_arrive_expect_tx(&bar[s], 0u); return; }
    rs_mbar_arrive_expect_tx(&bar[s], (unsigned)(SR * SW * 4));
    for (int b = 0; b < NB; ++b)  // NB boxes side by side: [SR][BW] each, stage layout [b][SR][BW]
      rs_tma_load_2d(buf + s * STAGE + b * BS, &map, c0 - PAD + b * BW, r0 - 1, &bar[s]);
  };
  if (tid == 0) {
    for (int q = 0; q < NSTAGE; ++q) rs_mbar_init(&bar[q], 1);
    rs_fence_barrier_init();
    for (int q = 0; q < NSTAGE - 1; ++q)
      if ((int)blockIdx.x + q * (int)gridDim.x < NTILES) issue(blockIdx.x + q * gridDim.x, q);
  }
  __syncthreads();
  int it = 0;
  for (int t = blockIdx.x; t < NTILES; t += gridDim.x, ++it) {
    const int s = it % NSTAGE;
    float* tile = buf + s * STAGE;
    if (tid == 0 && t + (NSTAGE - 1) * (int)gridDim.x < NTILES) {
      rs_bulk_wait_read_all();
      issue(t + (NSTAGE - 1) * gridDim.x, (it + NSTAGE - 1) % NSTAGE);
    }
    rs_mbar_wait(&bar[s], (unsigned)((it / NSTAGE) & 1));
    // each thread: 4 adjacent columns of TR*TC/1024 rows (interior), read then written back as [TR][TC]
    constexpr int CPR = TC / 4, ROWS_PER = TR * TC / 4 / 256;
    float4 v[ROWS_PER];
#pragma unroll
    for (int k = 0; k < ROWS_PER; ++k) {
      const int e = tid + k * 256, y = e / CPR, x = (e % CPR) * 4 + PAD;
      const int b = x / BW, xb = x % BW;
      v[k] = *reinterpret_cast<const float4*>(tile + b * BS + (y + 1) * BW + xb);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < ROWS_PER; ++k) {
      const int e = tid + k * 256, y = e / CPR, x = (e % CPR) * 4;
      constexpr int OB = TC < 256 ? TC : 256;  // store boxes of <= 256 columns: staging [TC/OB][TR][OB]
      *reinterpret_cast<float4*>(tile + (x / OB) * TR * OB + y * OB + x % OB) = v[k];
    }
    rs_fence_proxy_async();
    __syncthreads();
    if (tid == 0 && MODE != 1) {
      const int r0 = (t / NTX) * TR, c0 = (t % NTX) * TC;
      constexpr int OB = TC < 256 ? TC : 256;
      for (int b = 0; b < TC / OB; ++b) rs_tma_store_2d(&omap, c0 + b * OB, r0, tile + b * TR * OB);
      rs_bulk_commit();
    }
  }
  if (tid == 0) rs_bulk_wait_all();
}
"""


def main():
    import torch
    from paper_2201_03611_b200 import runtime as rt

    H = W = 8192
    sets = [(torch.rand(H * W, device="cuda"), torch.empty(H * W, device="cuda")) for _ in range(2)]
    sm = torch.cuda.get_device_properties(0).multi_processor_count
    stream = torch.cuda.current_stream()
    cfgs = [(64, 128, 1, 2, 3, 4, 0), (64, 128, 1, 2, 3, 4, 1), (64, 128, 1, 2, 3, 4, 2),
            (32, 256, 2, 2, 3, 4, 0), (32, 256, 2, 2, 3, 4, 1), (16, 512, 4, 2, 3, 8, 0),
            (16, 512, 4, 3, 2, 8, 0), (16, 512, 4, 2, 3, 8, 1), (8, 1024, 8, 2, 3, 8, 0)]
    for (TR, TC, NB, NS, BPS, PAD, MODE) in cfgs:
        SW = TC + 2 * PAD
        if SW % NB or SW // NB > 256 or (SW // NB) % 4:
            continue
        if W % TC or H % TR or (TR * TC // 4) % 256:
            continue
        SR = TR + 2
        stage = NB * (-(-(SR * (SW // NB)) // 32) * 32)
        smem = NS * stage * 4 + 8 * NS + 128
        if smem * BPS > 227 * 1024:
            continue
        name = f"tilecopy<{H}, {W}, {TR}, {TC}, {NB}, {NS}, {PAD}, {MODE}>"
        mod = rt.load_module(SRC, [name], ["--fmad=false"])
        fn = mod.function(mod.lowered[0])
        launches = []
        for src, dst in sets:
            m = rt.tma_desc_2d_f32(src.data_ptr(), W, H, W * 4, SW // NB, SR, 0)
            om = rt.tma_desc_2d_f32(dst.data_ptr(), W, H, W * 4, min(TC, 256), TR, 0)
            ntiles = (W // TC) * (H // TR)
            grid = min(ntiles, sm * BPS)
            launches.append(rt.PreparedLaunch(fn, (grid, 1, 1), (256, 1, 1),
                                              [ctypes.c_void_p(dst.data_ptr()), m, om], smem, stream))
        for i in range(6):
            launches[i % 2]()
        torch.cuda.synchronize()
        ok = torch.equal(sets[1][1], sets[1][0]) if MODE == 0 else None
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(40):
            launches[i % 2]()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 40
        nbytes = (2 if MODE == 0 else 1) * 4 * H * W
        print(f"TR={TR} TC={TC} boxes={NB} stages={NS} blocks/SM={BPS} mode={['copy', 'loads', 'stores'][MODE]}: "
              f"{ms * 1e3:.1f} us {nbytes / ms / 1e6:.0f} GB/s  exact={ok}", flush=True)


if __name__ == "__main__":
    main()
