#!/usr/bin/env python3
"""Data-movement probe for the 3x3 stencil: ROW STREAMING instead of tiles.

Each persistent block owns a contiguous band of output rows over the full
image width.  Whole input rows (W floats, one bulk copy each) stream through
a ring of NS shared-memory row slots, PF rows ahead; output row y is
computed from the slots of rows y-1, y, y+1 (clamped at the image edges,
padClamp) and leaves by 16-byte stores straight from registers.  DRAM sees
one long contiguous stream per block (reads) and one (writes); the only
re-read is the 2 halo rows per band.

The arithmetic is the CONV program's own order (bit-exact, packed fp32x2):
per window row  ((0 + w0*a0) + w1*a1) + w2*a2, then ((0 + r0) + r1) + r2.
Timed over two 256 MiB input sets round robin (> L2), steps back to back,
against torch's copy of the same bytes and checked bit-exact against a
torch restatement of the same order.

Measured (round 2, one B200; profiles/probe_rowstream_r02.txt): 101-117 us
per step against 92.5 us for the tiled stencil2d template and 85.8 us for
torch's copy of the same bytes — one row step per block at a time (three
mbarrier waits and a block barrier per 32 KiB row) loses to the tiled
template's independent tiles, so the template stays tiled."""
import ctypes
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

SRC = r"""
#include <rise/device.cuh>
template <int H, int W, int NT, int NS, int HALO_SHFL>
__global__ void __launch_bounds__(NT, 1) rowconv(float* __restrict__ out, const float* __restrict__ img,
                                                 const float* __restrict__ wgt) {
  constexpr int NCH = W / 4 / NT;  // float4 chunks per thread per row
  extern __shared__ __align__(128) unsigned char dsm[];
  float* slots = reinterpret_cast<float*>(dsm + ((128u - (rs_smem_addr(dsm) & 127u)) & 127u));
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(slots + NS * W);
  const int tid = threadIdx.x, lane = tid & 31;
  const int y0 = (int)((long long)blockIdx.x * H / gridDim.x);
  const int y1 = (int)((long long)(blockIdx.x + 1) * H / gridDim.x);
  const int lo = y0 > 0 ? y0 - 1 : 0, hi = y1 < H ? y1 : H - 1;  // input rows [lo, hi]
  float w[9];
#pragma unroll
  for (int e = 0; e < 9; ++e) w[e] = __ldg(wgt + e);
  int qi = 0;  // next input row (relative to lo) to issue; thread 0 only
  auto issue = [&](int q) {
    rs_fence_proxy_async();
    rs_mbar_arrive_expect_tx(&bar[q % NS], (unsigned)(W * 4));
    rs_bulk_g2s(slots + (q % NS) * W, img + (long long)(lo + q) * W, (unsigned)(W * 4), &bar[q % NS]);
  };
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) rs_mbar_init(&bar[s], 1);
    rs_fence_barrier_init();
    while (qi <= NS - 2 && lo + qi <= hi) issue(qi++);
  }
  __syncthreads();
  for (int y = y0; y < y1; ++y) {
    const int qa = (y > 0 ? y - 1 : 0) - lo, qb = y - lo, qc = (y < H - 1 ? y + 1 : H - 1) - lo;
    rs_mbar_wait(&bar[qa % NS], (unsigned)((qa / NS) & 1));
    rs_mbar_wait(&bar[qb % NS], (unsigned)((qb / NS) & 1));
    rs_mbar_wait(&bar[qc % NS], (unsigned)((qc / NS) & 1));
    const float* rows[3] = {slots + (qa % NS) * W, slots + (qb % NS) * W, slots + (qc % NS) * W};
#pragma unroll
    for (int j = 0; j < NCH; ++j) {
      const int c = 4 * (tid + j * NT);
      float a[3][6];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const float4 m = *reinterpret_cast<const float4*>(rows[i] + c);
        a[i][1] = m.x; a[i][2] = m.y; a[i][3] = m.z; a[i][4] = m.w;
        if (HALO_SHFL) {
          float l = __shfl_up_sync(0xffffffffu, m.w, 1), r = __shfl_down_sync(0xffffffffu, m.x, 1);
          if (lane == 0) l = rows[i][c > 0 ? c - 1 : 0];
          if (lane == 31) r = rows[i][c + 4 < W ? c + 4 : W - 1];
          a[i][0] = l; a[i][5] = r;
        } else {
          a[i][0] = rows[i][c > 0 ? c - 1 : 0];
          a[i][5] = rows[i][c + 4 < W ? c + 4 : W - 1];
        }
      }
      float o[4];
#pragma unroll
      for (int p = 0; p < 2; ++p) {  // output columns (2p, 2p+1) of the chunk, packed
        float2 t = make_float2(0.0f, 0.0f);
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          float2 s = __ffma2_rn(make_float2(a[i][2 * p], a[i][2 * p + 1]), make_float2(w[3 * i], w[3 * i]),
                                make_float2(0.0f, 0.0f));
          s = __fadd2_rn(s, __fmul2_rn(make_float2(a[i][2 * p + 1], a[i][2 * p + 2]),
                                       make_float2(w[3 * i + 1], w[3 * i + 1])));
          s = __fadd2_rn(s, __fmul2_rn(make_float2(a[i][2 * p + 2], a[i][2 * p + 3]),
                                       make_float2(w[3 * i + 2], w[3 * i + 2])));
          t = __fadd2_rn(t, s);
        }
        o[2 * p] = t.x; o[2 * p + 1] = t.y;
      }
      *reinterpret_cast<float4*>(out + (long long)y * W + c) = make_float4(o[0], o[1], o[2], o[3]);
    }
    __syncthreads();  // every read of the oldest slot is done
    if (tid == 0) {
      // slots may hold rows down to qc - 1 (the next output's first row)
      while (qi <= qc - 1 + NS - 1 && lo + qi <= hi) issue(qi++);
    }
  }
}
"""


def main():
    import torch
    from paper_2201_03611_b200 import runtime as rt

    H = W = 8192
    g = torch.Generator(device="cuda").manual_seed(3)
    sets = [(torch.rand(H * W, device="cuda", generator=g) * 2 - 1, torch.empty(H * W, device="cuda"))
            for _ in range(2)]
    wgt = torch.tensor([[1, 2, 1], [2, 4, 2], [1, 2, 1]], dtype=torch.float32, device="cuda") / 16
    sm = torch.cuda.get_device_properties(0).multi_processor_count
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    # reference in the program's order (elementwise fp32 ops are RN in torch)
    img = sets[1][0].view(H, W)
    p = torch.nn.functional.pad(img[None, None], (1, 1, 1, 1), mode="replicate")[0, 0]
    tot = torch.zeros(H, W, device="cuda")
    for i in range(3):
        s = torch.zeros(H, W, device="cuda")
        for j in range(3):
            s = s + p[i:i + H, j:j + W] * wgt[i, j]
        tot = tot + s
    ref = tot.reshape(-1)

    for _ in range(3):
        sets[0][1].copy_(sets[0][0])
    e0.record()
    for i in range(20):
        sets[i % 2][1].copy_(sets[i % 2][0])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"torch copy_ of the same bytes: {ms * 1e3:.1f} us {2 * 4 * H * W / ms / 1e6:.0f} GB/s", flush=True)

    # NS >= 4: rows y-1..y+1 in use while the next one is in flight
    for NT, NS, BPS, SHFL in [(512, 6, 1, 1), (512, 6, 1, 0), (1024, 6, 1, 1), (512, 5, 1, 1)]:
        smem = NS * W * 4 + 8 * NS + 128
        if smem * BPS > 227 * 1024 or (W // 4) % NT:
            continue
        name = f"rowconv<{H}, {W}, {NT}, {NS}, {SHFL}>"
        mod = rt.load_module(SRC, [name], ["--fmad=false"])
        fn = mod.function(mod.lowered[0])
        for grid in sorted({sm * BPS, sm * BPS - 2 * BPS}):
            launches = [rt.PreparedLaunch(fn, (grid, 1, 1), (NT, 1, 1),
                                          [ctypes.c_void_p(dst.data_ptr()), ctypes.c_void_p(src.data_ptr()),
                                           ctypes.c_void_p(wgt.data_ptr())], smem, stream)
                        for src, dst in sets]
            for i in range(6):
                launches[i % 2]()
            torch.cuda.synchronize()
            exact = torch.equal(sets[1][1], ref)
            e0.record()
            for i in range(40):
                launches[i % 2]()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 40
            nbytes = 4 * (2 * H * W + 9)
            print(f"NT={NT} NS={NS} blocks/SM={BPS} grid={grid} halo={'shfl' if SHFL else 'lds'}: "
                  f"{ms * 1e3:.1f} us {nbytes / ms / 1e6:.0f} GB/s exact={exact}", flush=True)


if __name__ == "__main__":
    main()
