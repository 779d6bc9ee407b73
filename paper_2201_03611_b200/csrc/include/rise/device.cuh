// rise/device.cuh — device helpers shared by every emitted sm_100a kernel.
// NVRTC-compiled (no host headers); included by the text emit_cuda produces.
#pragma once

#define RS_DEVICE __device__ __forceinline__

// padClamp index: min(max(k, 0), hi)  (extension.py semantics of padClamp)
RS_DEVICE int rs_clamp(int k, int hi) { return k < 0 ? 0 : (k > hi ? hi : k); }

// integer power for Pow sizes (the reference's ipow helper, codegen.py:38-44)
RS_DEVICE int rs_ipow(int base, int e) {
  int r = 1;
  while (e > 0) { r *= base; --e; }
  return r;
}

// IEEE binary32 reciprocal square root with both steps correctly rounded:
// bit-exact with the oracle definition rsqrt(x) = 1.0f / sqrt(x).
RS_DEVICE float rs_rsqrt_exact(float x) { return __fdiv_rn(1.0f, __fsqrt_rn(x)); }

// Fast path (MUFU.RSQ); used only where the program is compared under a
// tolerance (DESIGN.md parity rules).
RS_DEVICE float rs_rsqrt_fast(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// packed fp32x2 helpers (FFMA2 / FADD2 / FMUL2 are sm_100 instructions)
RS_DEVICE float2 rs_bcast2(float x) { return make_float2(x, x); }
RS_DEVICE float2 rs_neg2(float2 a) { return make_float2(-a.x, -a.y); }
RS_DEVICE float2 rs_div2(float2 a, float2 b) { return make_float2(a.x / b.x, a.y / b.y); }
RS_DEVICE float2 rs_rsqrt2(float2 a) { return make_float2(rs_rsqrt_fast(a.x), rs_rsqrt_fast(a.y)); }
RS_DEVICE float2 rs_sqrt2(float2 a) { return make_float2(sqrtf(a.x), sqrtf(a.y)); }
RS_DEVICE float2 rs_fabs2(float2 a) { return make_float2(fabsf(a.x), fabsf(a.y)); }
// correctly rounded per-lane forms for exact-mode packed bodies
//
// ptxas (CUDA 12.9) contracts mul.rn.f32x2 + add.rn.f32x2 into FFMA2 even
// with -fmad=false, which would break bit-exactness.  An exact packed
// product is therefore written fma(a, b, -0.0) with the -0.0 read from
// constant memory: equal to round(a * b) in every case (the -0.0 addend
// keeps +0/-0 products as they are), and ptxas cannot fold a following add
// into it because it cannot see the addend's value.
__constant__ float rs_negzero = -0.0f;
RS_DEVICE float2 rs_fmul2_exact(float2 a, float2 b) {
  return __ffma2_rn(a, b, make_float2(rs_negzero, rs_negzero));
}
RS_DEVICE float2 rs_div2_rn(float2 a, float2 b) { return make_float2(__fdiv_rn(a.x, b.x), __fdiv_rn(a.y, b.y)); }
RS_DEVICE float2 rs_sqrt2_rn(float2 a) { return make_float2(__fsqrt_rn(a.x), __fsqrt_rn(a.y)); }
RS_DEVICE float2 rs_rsqrt2_rn(float2 a) { return make_float2(rs_rsqrt_exact(a.x), rs_rsqrt_exact(a.y)); }

RS_DEVICE unsigned rs_smem_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// ---- mbarrier / bulk-copy (TMA) primitives ---------------------------------

RS_DEVICE void rs_mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(rs_smem_addr(bar)), "r"(count) : "memory");
}

RS_DEVICE void rs_fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

RS_DEVICE void rs_fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

RS_DEVICE void rs_mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(rs_smem_addr(bar)),
               "r"(bytes)
               : "memory");
}

RS_DEVICE void rs_mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(rs_smem_addr(bar)) : "memory");
}

RS_DEVICE bool rs_mbar_try_wait(unsigned long long* bar, unsigned phase) {
  unsigned ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(rs_smem_addr(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}

RS_DEVICE void rs_mbar_wait(unsigned long long* bar, unsigned phase) {
  while (!rs_mbar_try_wait(bar, phase)) {
  }
}

// 1-D bulk copy global -> shared (TMA engine), completion counted in bytes on
// `bar`.  src, dst and bytes must be multiples of 16.
RS_DEVICE void rs_bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          rs_smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(rs_smem_addr(bar))
      : "memory");
}

// A CUtensorMap passed by value as a __grid_constant__ kernel parameter.
struct alignas(64) rs_tmap {
  unsigned long long words[16];
};

RS_DEVICE void rs_tmap_prefetch(const rs_tmap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<unsigned long long>(map)) : "memory");
}

// 2-D TMA tile load (coordinates: inner c0, outer c1) into shared memory,
// completion counted in bytes on `bar`.
RS_DEVICE void rs_tma_load_2d(void* dst, const rs_tmap* map, int c0, int c1, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          rs_smem_addr(dst)),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(rs_smem_addr(bar))
      : "memory");
}

// 2-D TMA tile store shared -> global (out-of-range box elements are not
// written), tracked as a bulk async-group of the issuing thread.
RS_DEVICE void rs_tma_store_2d(const rs_tmap* map, int c0, int c1, const void* src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<unsigned long long>(map)),
               "r"(c0), "r"(c1), "r"(rs_smem_addr(src))
               : "memory");
}
// 1-D bulk copy shared -> global (16-byte aligned, size a multiple of 16),
// tracked as a bulk async-group of the issuing thread.
RS_DEVICE void rs_bulk_s2g(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                   reinterpret_cast<unsigned long long>(dst)),
               "r"(rs_smem_addr(src)), "r"(bytes)
               : "memory");
}
RS_DEVICE void rs_bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// the shared-memory sources of every committed bulk store have been read
RS_DEVICE void rs_bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
// every committed bulk store has completed
RS_DEVICE void rs_bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// 128-bit streaming global load that does not allocate in L1.
RS_DEVICE float4 rs_ldg_stream(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

// Grid-wide barrier for kernels launched cooperatively (RS_LAUNCH_COOPERATIVE:
// every block co-resident).  bar[0] counts arrivals, bar[1] is the
// generation; both start at 0 (a zeroed workspace) and bar[0] returns to 0.
RS_DEVICE void rs_grid_sync(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = bar + 1;
    const unsigned g = *gen;  // read before arriving: the last arrival may bump it
    __threadfence();          // this block's writes before its arrival
    if (atomicAdd(bar, 1u) == gridDim.x * gridDim.y * gridDim.z - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g) __nanosleep(64);
    }
    __threadfence();  // everyone's writes before this block continues
  }
  __syncthreads();
}

// Cross-GPU exchange slot (peer memory, system scope): a 64-bit word
// (epoch << 32 | payload bits).  rs_xchg_put publishes a value for `epoch`;
// rs_xchg_get spins until the slot holds `epoch` and returns the payload.
// A rank that never arrives traps after ~20 s instead of hanging the GPU.
RS_DEVICE void rs_xchg_put(unsigned long long* slot, unsigned epoch, unsigned payload) {
  const unsigned long long v = ((unsigned long long)epoch << 32) | payload;
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(slot), "l"(v) : "memory");
}
RS_DEVICE unsigned rs_xchg_get(const unsigned long long* slot, unsigned epoch) {
  unsigned long long v, t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(slot) : "memory");
    if ((unsigned)(v >> 32) == epoch) return (unsigned)v;
    __nanosleep(100);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 20000000000ull) __trap();  // a peer never published: fail loudly
  }
}

// Epoch-tagged 64-bit slot inside one GPU (epoch << 32 | payload bits): one
// relaxed store publishes tag and payload together (single-copy atomic), so
// neither side needs a fence; the reader spins until the slot carries its
// epoch.  A launch that never publishes makes the reader trap after ~20 s.
RS_DEVICE void rs_slot_put(unsigned long long* slot, unsigned epoch, unsigned payload) {
  const unsigned long long v = ((unsigned long long)epoch << 32) | payload;
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(slot), "l"(v) : "memory");
}
RS_DEVICE unsigned rs_slot_get(const unsigned long long* slot, unsigned epoch) {
  unsigned long long v, t0, t;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(slot) : "memory");
  if ((unsigned)(v >> 32) == epoch) return (unsigned)v;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    __nanosleep(32);
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(slot) : "memory");
    if ((unsigned)(v >> 32) == epoch) return (unsigned)v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 20000000000ull) __trap();
  }
}

RS_DEVICE unsigned rs_lane() { return threadIdx.x & 31u; }
RS_DEVICE unsigned rs_warp() { return threadIdx.x >> 5; }
