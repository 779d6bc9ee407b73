// Dependent-fold latency on one B200 (diagnostic for rowfold's per-row
// floor): ONE warp per SM sub-partition folds acc = acc + a[j] * x[j] in j
// order (round-to-nearest multiply then add, no contraction: the exact
// program order) over N columns, with operands from registers or from
// shared memory; prints cycles per column.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe_chain tools/probe_chain.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 8192;

template <int MODE>
__global__ void __launch_bounds__(128) fold(float* out, float s) {
  __shared__ __align__(16) float sa[2048], sx[2048];
  for (int e = threadIdx.x; e < 2048; e += 128) { sa[e] = s * e; sx[e] = 1.0f - s * e; }
  __syncthreads();
  float acc = 0.0f, acc2 = 0.0f;
  const float a0 = s * threadIdx.x, x0 = 1.0f - s;
  long long t0 = clock64();
  if (MODE == 0) {  // operands in registers
#pragma unroll 16
    for (int j = 0; j < N; ++j) acc = __fadd_rn(acc, __fmul_rn(a0 + j, x0));
  } else if (MODE == 1) {  // operands from shared memory, float4 per 4 columns
#pragma unroll 16
    for (int j = 0; j < N; j += 4) {
      const float4 a = *reinterpret_cast<const float4*>(sa + ((j + 4 * threadIdx.x) & 2047));
      const float4 x = *reinterpret_cast<const float4*>(sx + (j & 2047));
      acc = __fadd_rn(acc, __fmul_rn(a.x, x.x));
      acc = __fadd_rn(acc, __fmul_rn(a.y, x.y));
      acc = __fadd_rn(acc, __fmul_rn(a.z, x.z));
      acc = __fadd_rn(acc, __fmul_rn(a.w, x.w));
    }
  } else if (MODE == 2) {  // plain dependent FADD chain (no multiply)
#pragma unroll 16
    for (int j = 0; j < N; ++j) acc = __fadd_rn(acc, a0 + j);
  } else {  // two independent rows per lane (the chains interleave)
#pragma unroll 16
    for (int j = 0; j < N; ++j) {
      acc = __fadd_rn(acc, __fmul_rn(a0 + j, x0));
      acc2 = __fadd_rn(acc2, __fmul_rn(a0 - j, x0));
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (float)(t1 - t0);
  if (acc + acc2 == 1234.5f) out[0] = acc;
}

template <int MODE>
void run(const char* name) {
  float *d, h[2];
  cudaMalloc(&d, 8);
  fold<MODE><<<148, 128>>>(d, 0.001f);
  fold<MODE><<<148, 128>>>(d, 0.001f);
  cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
  printf("%-44s %6.2f cycles per column (clock64, block 0)\n", name, h[1] / N);
  cudaFree(d);
}

int main() {
  run<0>("fold a*x, operands in registers");
  run<1>("fold a*x, float4 operands from shared memory");
  run<2>("plain dependent FADD chain");
  run<3>("two rows per lane (two chains)");
  return 0;
}
