// Packed-FP32 issue ceiling on one B200 (diagnostic for the allpairs bound):
// throughput of FFMA2 / FMUL2 / FADD2 in their register / broadcast /
// immediate operand forms, of the nbody pair body without and with its
// MUFU rsqrt, and of scalar FFMA, each as lane-operations per SM per clock
// (the FP32 peak is 128).  Build: nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -o probe_fp32x2 tools/probe_fp32x2.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CH = 8;      // independent chains per thread
constexpr int IT = 4096;   // iterations

__device__ __forceinline__ float ex2_approx(float v) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}
__device__ __forceinline__ float lg2_approx(float v) {
  float r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) k(float* out, float s) {
  float2 a[CH], b[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    a[c] = make_float2(threadIdx.x * 1e-3f + c, s * c);
    b[c] = make_float2(s + c, 1.0f - c * s);
  }
  const float2 m = make_float2(s, s * 0.5f);
  float x = s;
  for (int i = 0; i < IT; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (MODE == 0) a[c] = __ffma2_rn(a[c], b[c], a[c]);                    // r, r, r
      if (MODE == 1) a[c] = __ffma2_rn(a[c], a[c], make_float2(0.01f, 0.01f));  // r, r, imm
      if (MODE == 2) a[c] = __fmul2_rn(a[c], b[c]);                          // r, r
      if (MODE == 3) a[c] = __fadd2_rn(make_float2(x, x), a[c]);             // broadcast, r
      if (MODE == 4) { a[c].x = fmaf(a[c].x, b[c].x, a[c].y); a[c].y = fmaf(a[c].y, b[c].y, a[c].x); }  // scalar FFMA
      if (MODE == 8) { a[c].x = rsqrtf(a[c].x); a[c].y = rsqrtf(a[c].y); }  // MUFU only
      if (MODE == 10) {  // one FFMA2 + one ALU-pipe LOP3 per chain step
        a[c] = __ffma2_rn(a[c], b[c], a[c]);
        b[c].x = __int_as_float(__float_as_int(b[c].x) ^ (i & 1));
      }
      if (MODE == 11) {  // one packed FFMA2 and one independent scalar FFMA per chain step
        a[c] = __ffma2_rn(a[c], b[c], a[c]);
        b[c].x = fmaf(b[c].x, x, b[c].y);
      }
      if (MODE == 12) {  // one packed FFMA2 and two independent scalar FFMAs per chain step
        a[c] = __ffma2_rn(a[c], b[c], a[c]);
        b[c].x = fmaf(b[c].x, x, 0.5f);
        b[c].y = fmaf(b[c].y, x, 0.25f);
      }
      if (MODE == 13) { a[c].x = ex2_approx(a[c].x); a[c].y = ex2_approx(a[c].y); }  // MUFU.EX2 only
      if (MODE == 14) { a[c].x = lg2_approx(a[c].x); a[c].y = lg2_approx(a[c].y); }  // MUFU.LG2 only
      if (MODE == 15) {
        // the pair body with s = m r^-3 as ex2(log2 m - 1.5 log2 r2): one FFMA2 and
        // 2 + 2 MUFU (LG2, EX2) in place of 3 FMUL2 and 2 MUFU.RSQ
        float2 d = __fadd2_rn(make_float2(x, x), make_float2(-a[c].x, -a[c].y));
        float2 r2 = __ffma2_rn(d, d, make_float2(0.01f, 0.01f));
        r2 = __ffma2_rn(d, d, r2);
        r2 = __ffma2_rn(d, d, r2);
        float2 l = make_float2(lg2_approx(r2.x), lg2_approx(r2.y));
        l = __ffma2_rn(l, make_float2(-1.5f, -1.5f), m);
        float2 q2 = make_float2(ex2_approx(l.x), ex2_approx(l.y));
        b[c] = __ffma2_rn(d, q2, b[c]);
        b[c] = __ffma2_rn(d, q2, b[c]);
        b[c] = __ffma2_rn(d, q2, b[c]);
        a[c].x += 1e-7f;
      }
      if (MODE == 5 || MODE == 6 || MODE == 7 || MODE == 9) {
        // the nbody pair body for two targets (12 packed FP32 ops): a = target
        // position component, b = accumulator; x, m = source scalars
        float2 d = __fadd2_rn(make_float2(x, x), make_float2(-a[c].x, -a[c].y));
        float2 r2 = __ffma2_rn(d, d, make_float2(0.01f, 0.01f));
        r2 = __ffma2_rn(d, d, r2);
        r2 = __ffma2_rn(d, d, r2);
        float2 q = MODE == 6 ? make_float2(rsqrtf(r2.x), rsqrtf(r2.y))
                 : MODE == 7 ? make_float2(rsqrtf(r2.x), r2.y)
                 : MODE == 9 ? make_float2(__int_as_float(__float_as_int(r2.x) ^ 0x5f3759df),
                                           __int_as_float(__float_as_int(r2.y) ^ 0x5f3759df)) : r2;
        float2 q2 = __fmul2_rn(q, q);
        q2 = __fmul2_rn(q2, q);
        q2 = __fmul2_rn(m, q2);
        b[c] = __ffma2_rn(d, q2, b[c]);
        b[c] = __ffma2_rn(d, q2, b[c]);
        b[c] = __ffma2_rn(d, q2, b[c]);
        a[c].x += 1e-7f;  // keep the chains live
      }
    }
    x += 1e-6f;
  }
  float t = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) t += a[c].x + a[c].y + b[c].x + b[c].y;
  if (t == 1234.5f) out[0] = t;
}

template <int MODE>
void run(const char* name, double lane_ops_per_chain_iter, int blocks_per_sm) {
  int dev = 0, sms = 0, clk_khz = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  float* out;
  cudaMalloc(&out, 4);
  dim3 grid(sms * blocks_per_sm), block(512);
  k<MODE><<<grid, block>>>(out, 0.5f);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k<MODE><<<grid, block>>>(out, 0.5f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  double ops = 5.0 * grid.x * block.x * (double)IT * CH * lane_ops_per_chain_iter;
  double per_sm_clk = ops / (ms * 1e-3) / sms / (clk_khz * 1e3);
  printf("%-34s %8.3f ms  %7.1f lane-ops/SM/clk (max clock %d MHz)\n", name, ms, per_sm_clk, clk_khz / 1000);
  cudaFree(out);
}

int main() {
  run<0>("FFMA2 r,r,r", 2, 1);
  run<1>("FFMA2 r,r,imm", 2, 1);
  run<2>("FMUL2 r,r", 2, 1);
  run<3>("FADD2 bcast,r", 2, 1);
  run<4>("FFMA r,r,r (scalar, 2 per chain)", 2, 1);
  run<5>("nbody body, no MUFU (24 per chain)", 24, 1);
  run<6>("nbody body with MUFU (24 per chain)", 24, 1);
  run<7>("nbody body, 1 MUFU per 2 pairs", 24, 1);
  run<8>("MUFU.RSQ only (2 per chain)", 2, 1);
  run<9>("nbody body, 2 ALU ops for the MUFU", 24, 1);
  run<10>("FFMA2 + LOP3 (FFMA2 lanes only)", 2, 1);
  run<11>("FFMA2 + scalar FFMA (3 lanes per chain)", 3, 1);
  run<12>("FFMA2 + 2 scalar FFMA (4 per chain)", 4, 1);
  run<13>("MUFU.EX2 only (2 per chain)", 2, 1);
  run<14>("MUFU.LG2 only (2 per chain)", 2, 1);
  run<15>("nbody body via LG2/EX2 (24 per chain)", 24, 1);
  return 0;
}
