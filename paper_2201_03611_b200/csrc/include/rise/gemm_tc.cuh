// rise/gemm_tc.cuh — fp32 GEMM on the 5th-generation tensor cores (tcgen05)
// with the 3xTF32 split, for the `gemm_tc` template (tmpl_gemm.py).
//
//   C[M x N] = A[M x K] * Bt[N x K]^T      (both operands K-major)
//
// 3xTF32: x = hi + lo with hi = x with the low 13 mantissa bits cleared
// (exactly representable in TF32) and lo = x - hi (exact in fp32).  Then
//   A*B ~= A_hi*B_hi + A_hi*B_lo + A_lo*B_hi
// (the dropped A_lo*B_lo and the TF32 rounding of lo are ~2^-22 relative),
// accumulated in fp32 in tensor memory: fp32-level accuracy at TF32 speed.
//
// CTA tile 128 x BN, K step 32 (one 128-byte swizzle atom), STAGES-deep ring:
//   warp 0      TMA producer: raw fp32 A / B tiles -> shared memory (SW128)
//   warp 1      TMEM allocator + MMA issuer (one elected thread): 12
//               tcgen05.mma.kind::tf32 (M=128, N=BN, K=8) per stage into a
//               BN-column fp32 TMEM accumulator; tcgen05.commit frees stages
//   warps 2..5  split each landed stage (raw -> hi in place unless the
//               tensor core already ignores the low 13 bits, new lo tiles),
//               then the epilogue: tcgen05.ld 32x32b -> registers -> global
#pragma once
#include "device.cuh"

namespace rise_gemm {

constexpr int BM = 128, BK = 32;

template <int BN_, int STAGES_>
struct Cfg {
  static constexpr int BN = BN_;
  static constexpr int STAGES = STAGES_;
  static constexpr int TILE_A = BM * BK * 4;  // 16 KiB
  static constexpr int TILE_B = BN * BK * 4;  // 16 or 32 KiB
  static constexpr int STAGE_BYTES = 2 * (TILE_A + TILE_B);
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr unsigned TMEM_COLS = BN;
  // instruction descriptor, kind::tf32: D f32 (bits 4-5 = 1), A/B tf32
  // (bits 7-9, 10-12 = 2), both K-major (bits 15, 16 = 0), N >> 3 at bit 17,
  // M >> 4 at bit 24
  static constexpr unsigned IDESC =
      (1u << 4) | (2u << 7) | (2u << 10) | (unsigned(BN >> 3) << 17) | (unsigned(BM >> 4) << 24);
};

constexpr int THREADS = 192;

// shared-memory matrix descriptor, K-major, 128-byte swizzle: start >> 4,
// LBO = 1 (unused for swizzled K-major), SBO = 1024 B (8 rows x 128 B) >> 4,
// version 1 (sm_100), layout type 2 (SWIZZLE_128B)
RS_DEVICE unsigned long long smem_desc(unsigned saddr) {
  unsigned long long d = (unsigned long long)((saddr >> 4) & 0x3FFFu);
  d |= 1ull << 16;
  d |= (unsigned long long)(1024 >> 4) << 32;
  d |= 1ull << 46;
  d |= 2ull << 61;
  return d;
}

template <unsigned IDESC>
RS_DEVICE void mma(unsigned tmem_d, unsigned long long adesc, unsigned long long bdesc, unsigned accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(IDESC), "r"(accumulate));
}

RS_DEVICE void commit(unsigned long long* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   rs_smem_addr(bar))
               : "memory");
}

RS_DEVICE void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
RS_DEVICE void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

template <unsigned COLS>
RS_DEVICE void tmem_alloc(unsigned* slot) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(rs_smem_addr(slot)),
               "r"(COLS)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

template <unsigned COLS>
RS_DEVICE void tmem_dealloc(unsigned taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(COLS) : "memory");
}

// 32 consecutive fp32 columns of this warp's 32 TMEM lanes -> 32 registers
RS_DEVICE void tmem_ld32(unsigned taddr, unsigned* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

RS_DEVICE float4 split_hi(float4 v) {
  return make_float4(__uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u),
                     __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u),
                     __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u),
                     __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u));
}

template <bool WRITE_HI>
RS_DEVICE void split_tile(unsigned char* raw, unsigned char* lo, int bytes, int t) {
  float4* r = reinterpret_cast<float4*>(raw);
  float4* l = reinterpret_cast<float4*>(lo);
#pragma unroll 4
  for (int i = t; i < bytes / 16; i += 128) {
    const float4 v = r[i];
    const float4 h = split_hi(v);
    if (WRITE_HI) r[i] = h;
    l[i] = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
  }
}

// C (row pitch ldc) for the 128 x BN tile at (blockIdx.y, blockIdx.x)
template <int K, int BN, int STAGES, bool WRITE_HI>
RS_DEVICE void gemm_3xtf32(float* __restrict__ C, int ldc, const rs_tmap* mapA, const rs_tmap* mapB) {
  using G = Cfg<BN, STAGES>;
  extern __shared__ __align__(1024) unsigned char rs_gemm_smem_raw[];
  unsigned char* smem =
      rs_gemm_smem_raw + ((1024u - (rs_smem_addr(rs_gemm_smem_raw) & 1023u)) & 1023u);
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem + STAGES * G::STAGE_BYTES);
  unsigned long long* full = bars;
  unsigned long long* conv = bars + STAGES;
  unsigned long long* empty = bars + 2 * STAGES;
  unsigned long long* tmem_full = bars + 3 * STAGES;
  unsigned* tmem_slot = reinterpret_cast<unsigned*>(bars + 3 * STAGES + 1);

  constexpr int KB = K / BK;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  auto a_raw = [&](int s) { return smem + s * G::STAGE_BYTES; };
  auto a_lo = [&](int s) { return smem + s * G::STAGE_BYTES + G::TILE_A; };
  auto b_raw = [&](int s) { return smem + s * G::STAGE_BYTES + 2 * G::TILE_A; };
  auto b_lo = [&](int s) { return smem + s * G::STAGE_BYTES + 2 * G::TILE_A + G::TILE_B; };

  if (threadIdx.x == 0) {
    rs_tmap_prefetch(mapA);
    rs_tmap_prefetch(mapB);
    for (int s = 0; s < STAGES; ++s) {
      rs_mbar_init(&full[s], 1);
      rs_mbar_init(&conv[s], 4);
      rs_mbar_init(&empty[s], 1);
    }
    rs_mbar_init(tmem_full, 1);
    rs_fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<G::TMEM_COLS>(tmem_slot);
  fence_before();
  __syncthreads();
  fence_after();
  const unsigned tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < KB; ++kb) {
        const int s = kb % STAGES;
        const unsigned ph = (unsigned)((kb / STAGES) & 1);
        rs_mbar_wait(&empty[s], ph ^ 1u);
        rs_mbar_arrive_expect_tx(&full[s], G::TILE_A + G::TILE_B);
        rs_tma_load_2d(a_raw(s), mapA, kb * BK, m0, &full[s]);
        rs_tma_load_2d(b_raw(s), mapB, kb * BK, n0, &full[s]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      for (int kb = 0; kb < KB; ++kb) {
        const int s = kb % STAGES;
        const unsigned ph = (unsigned)((kb / STAGES) & 1);
        rs_mbar_wait(&full[s], ph);
        rs_mbar_wait(&conv[s], ph);
        fence_after();
        const unsigned long long ahi = smem_desc(rs_smem_addr(a_raw(s)));
        const unsigned long long alo = smem_desc(rs_smem_addr(a_lo(s)));
        const unsigned long long bhi = smem_desc(rs_smem_addr(b_raw(s)));
        const unsigned long long blo = smem_desc(rs_smem_addr(b_lo(s)));
#pragma unroll
        for (int k = 0; k < BK / 8; ++k) {
          const unsigned long long off = (unsigned long long)(k * 32) >> 4;  // 8 tf32 = 32 bytes
          mma<G::IDESC>(tmem, alo + off, bhi + off, (kb | k) != 0);
          mma<G::IDESC>(tmem, ahi + off, blo + off, 1u);
          mma<G::IDESC>(tmem, ahi + off, bhi + off, 1u);
        }
        commit(&empty[s]);
      }
      commit(tmem_full);
    }
    __syncwarp();
  } else {
    const int t = threadIdx.x - 64;
    for (int kb = 0; kb < KB; ++kb) {
      const int s = kb % STAGES;
      const unsigned ph = (unsigned)((kb / STAGES) & 1);
      rs_mbar_wait(&full[s], ph);
      split_tile<WRITE_HI>(a_raw(s), a_lo(s), G::TILE_A, t);
      split_tile<WRITE_HI>(b_raw(s), b_lo(s), G::TILE_B, t);
      rs_fence_proxy_async();
      __syncwarp();
      if (lane == 0) rs_mbar_arrive(&conv[s]);
    }
    // epilogue: TMEM lanes [32q, 32q+32) belong to warp (q mod 4)
    rs_mbar_wait(tmem_full, 0u);
    fence_after();
    const int q = warp & 3;
    const int row = q * 32 + lane;
    float* crow = C + (long long)(m0 + row) * ldc + n0;
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
      unsigned r[32];
      tmem_ld32(tmem + ((unsigned)(q * 32) << 16) + (unsigned)c0, r);
#pragma unroll
      for (int j = 0; j < 32; j += 4) {
        *reinterpret_cast<float4*>(crow + c0 + j) =
            make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]), __uint_as_float(r[j + 2]),
                        __uint_as_float(r[j + 3]));
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 1) {
    fence_after();
    tmem_dealloc<G::TMEM_COLS>(tmem);
  }
}

// ---------------------------------------------------------------------------
// CTA-pair variant (tcgen05 cta_group::2): a cluster of two CTAs on a TPC
// computes a 256 x BN tile with M=256 MMAs issued by the leader CTA.  Each CTA
// stages its own 128 rows of A and BN/2 rows of Bt (raw + lo), so every byte
// of shared memory feeds twice the MMA work of the single-CTA kernel; the
// accumulator rows 0-127 live in the leader's TMEM, 128-255 in the peer's.
//
//   both CTAs, warp 0   TMA of the CTA's own A / Bt halves (local barrier)
//   both CTAs, warp 1   tcgen05.alloc.cta_group::2; leader lane 0 issues the
//                       MMAs and multicasts tcgen05.commit to both CTAs
//   both CTAs, 2..5     split hi/lo in place, then arrive (cluster scope) on
//                       the LEADER's conv barrier; epilogue from own TMEM

RS_DEVICE unsigned cluster_ctarank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

RS_DEVICE unsigned mapa(unsigned saddr, unsigned rank) {
  unsigned out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(saddr), "r"(rank));
  return out;
}

RS_DEVICE void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// 16-byte async-proxy copy into the peer CTA's shared memory whose
// completion is a complete_tx on the peer's mbarrier: the cross-CTA "stage
// converted" signal.  The copy is issued after fence.proxy.async + a barrier
// of the converting threads and its complete_tx has release semantics, so
// it orders those threads' shared-memory writes before the peer's MMA reads
// (an acquire wait) without a cluster-scope MEMBAR in the instruction stream.
RS_DEVICE void signal_s2s_cluster(unsigned dst_cluster_addr, const void* src, unsigned bar_cluster_addr) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];" ::"r"(
          dst_cluster_addr),
      "r"(rs_smem_addr(src)), "r"(bar_cluster_addr)
      : "memory");
}

RS_DEVICE void mbar_arrive_remote(unsigned cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

RS_DEVICE void mbar_wait_cluster(unsigned long long* bar, unsigned phase) {
  unsigned ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(rs_smem_addr(bar)), "r"(phase)
        : "memory");
  }
}

// the instruction descriptor is a register operand: one kernel issues both
// full (N = BN) and half-width (N = BN / 2) tiles
RS_DEVICE void mma2(unsigned tmem_d, unsigned long long adesc, unsigned long long bdesc, unsigned idesc,
                    unsigned accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

RS_DEVICE void commit2_multicast(unsigned long long* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          rs_smem_addr(bar)),
      "h"((unsigned short)3)
      : "memory");
}

template <unsigned COLS>
RS_DEVICE void tmem_alloc2(unsigned* slot) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(rs_smem_addr(slot)),
               "r"(COLS)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}

template <unsigned COLS>
RS_DEVICE void tmem_dealloc2(unsigned taddr) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(COLS) : "memory");
}

// MN-major variant (B stored K x N, row-major).  MN-major tf32 operands
// only exist in the 128-byte swizzle with 32-byte atomicity (UMMA layout
// type 1, SWIZZLE_128B_BASE32B; the TMA map uses
// CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B): atoms of 4 K-rows x 32 N-values
// (512 B); consecutive 32-column N groups are LBO = 4 KiB apart (one 32 x 32
// TMA box each), K atoms SBO = 512 B apart.
RS_DEVICE unsigned long long smem_desc_mn(unsigned saddr) {
  unsigned long long d = (unsigned long long)((saddr >> 4) & 0x3FFFu);
  d |= (unsigned long long)(4096 >> 4) << 16;
  d |= (unsigned long long)(512 >> 4) << 32;
  d |= 1ull << 46;
  d |= 1ull << 61;
  return d;
}

template <int BN_, int STAGES_>
struct Cfg2 {
  static constexpr int BN = BN_;  // pair tile: 256 x BN; each CTA stages BN/2 rows of Bt
  static constexpr int STAGES = STAGES_;
  static constexpr int TILE_A = 128 * BK * 4;
  static constexpr int TILE_B = (BN / 2) * BK * 4;
  static constexpr int STAGE_BYTES = 2 * (TILE_A + TILE_B);
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;
  static constexpr unsigned TMEM_COLS = BN;
  static constexpr unsigned IDESC =
      (1u << 4) | (2u << 7) | (2u << 10) | (unsigned(BN >> 3) << 17) | (unsigned(256 >> 4) << 24);
  static constexpr unsigned IDESC_HALF =
      (1u << 4) | (2u << 7) | (2u << 10) | (unsigned((BN / 2) >> 3) << 17) | (unsigned(256 >> 4) << 24);
  static constexpr unsigned IDESC_BMN = IDESC | (1u << 16);  // b_major = MN
};

// blockIdx.x = 2 * pair + rank.  Tiles 256 x BN in (tm, tn) order, tn
// fastest.  Pairs below n_full each compute one whole tile.  The tiles after
// them (the tail that would leave most SM pairs idle in a last partial wave:
// 256 tiles on 74 pairs are 3.46 waves) are split along K: pair n_full + 2u
// folds the first half of tile n_full + u's K loop, pair n_full + 2u + 1 the
// second half, which it parks in `ws`; the first-half pair waits for it
// (flag, release / acquire) and stores C = first + second.  Every split unit
// is resident at once (the split is only used when the units fit in one
// wave), the second half never waits, and the order of the final add is
// fixed: deterministic.
template <int M, int N, int K, int BN, int STAGES, bool B_MN = false>
RS_DEVICE void gemm_3xtf32_2sm(float* __restrict__ C, int ldc, const rs_tmap* mapA, const rs_tmap* mapB,
                               int n_full, float* __restrict__ ws, unsigned* __restrict__ flags) {
  using G = Cfg2<BN, STAGES>;
  extern __shared__ __align__(1024) unsigned char rs_gemm_smem_raw[];
  unsigned char* smem =
      rs_gemm_smem_raw + ((1024u - (rs_smem_addr(rs_gemm_smem_raw) & 1023u)) & 1023u);
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem + STAGES * G::STAGE_BYTES);
  unsigned long long* full = bars;
  unsigned long long* conv = bars + STAGES;
  unsigned long long* empty = bars + 2 * STAGES;
  unsigned long long* tmem_full = bars + 3 * STAGES;
  unsigned* tmem_slot = reinterpret_cast<unsigned*>(bars + 3 * STAGES + 1);
  // 16-byte landing slot of the CTA-1 -> CTA-0 "stage converted" signal copies
  unsigned char* sig_slot = reinterpret_cast<unsigned char*>(bars) + ((3 * STAGES + 2) * 8 + 15) / 16 * 16;

  // ragged shapes: the TMA unit zero-fills the parts of the edge tiles
  // outside A / B (a zero K tail adds nothing), and the epilogue stores only
  // in-range rows and columns
  constexpr int KB = (K + BK - 1) / BK;
  constexpr int NTN = (N + BN - 1) / BN;
  const unsigned rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1;
  const bool split = pair >= n_full;
  const int unit = pair - n_full;  // split units only
  const int tile = split ? n_full + (unit >> 1) : pair;
  const int khalf = split ? (unit & 1) : 0;
  const int kb0 = split && khalf ? KB / 2 : 0;
  const int kb1 = split && !khalf ? KB / 2 : KB;
  const int m0 = (tile / NTN) * 256, n0 = (tile % NTN) * BN;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto a_raw = [&](int s) { return smem + s * G::STAGE_BYTES; };
  auto a_lo = [&](int s) { return smem + s * G::STAGE_BYTES + G::TILE_A; };
  auto b_raw = [&](int s) { return smem + s * G::STAGE_BYTES + 2 * G::TILE_A; };
  auto b_lo = [&](int s) { return smem + s * G::STAGE_BYTES + 2 * G::TILE_A + G::TILE_B; };

  if (threadIdx.x == 0) {
    rs_tmap_prefetch(mapA);
    rs_tmap_prefetch(mapB);
    for (int s = 0; s < STAGES; ++s) {
      rs_mbar_init(&full[s], 1);
      // phase = CTA 0's converters (one arrival, +16 tx expected) and CTA 1's
      // signal copy (complete_tx 16 bytes), in either order
      rs_mbar_init(&conv[s], 1);
      rs_mbar_init(&empty[s], 1);
    }
    rs_mbar_init(tmem_full, 1);
    rs_fence_barrier_init();
  }
  if (warp == 1) tmem_alloc2<G::TMEM_COLS>(tmem_slot);
  fence_before();
  cluster_sync();
  fence_after();
  const unsigned tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = kb0; kb < kb1; ++kb) {
        const int s = (kb - kb0) % STAGES;
        const unsigned ph = (unsigned)(((kb - kb0) / STAGES) & 1);
        rs_mbar_wait(&empty[s], ph ^ 1u);
        rs_mbar_arrive_expect_tx(&full[s], G::TILE_A + G::TILE_B);
        rs_tma_load_2d(a_raw(s), mapA, kb * BK, m0 + 128 * (int)rank, &full[s]);
        if (B_MN) {  // BN/2 columns of K x N B as 32 x 32 boxes, 4 KiB apart
#pragma unroll
          for (int b = 0; b < BN / 64; ++b)
            rs_tma_load_2d(b_raw(s) + b * 4096, mapB, n0 + (BN / 2) * (int)rank + 32 * b, kb * BK, &full[s]);
        } else {
          rs_tma_load_2d(b_raw(s), mapB, kb * BK, n0 + (BN / 2) * (int)rank, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0 && lane == 0) {
      for (int kb = kb0; kb < kb1; ++kb) {
        const int s = (kb - kb0) % STAGES;
        const unsigned ph = (unsigned)(((kb - kb0) / STAGES) & 1);
        mbar_wait_cluster(&conv[s], ph);
        fence_after();
        const unsigned long long ahi = smem_desc(rs_smem_addr(a_raw(s)));
        const unsigned long long alo = smem_desc(rs_smem_addr(a_lo(s)));
        const unsigned long long bhi =
            B_MN ? smem_desc_mn(rs_smem_addr(b_raw(s))) : smem_desc(rs_smem_addr(b_raw(s)));
        const unsigned long long blo =
            B_MN ? smem_desc_mn(rs_smem_addr(b_lo(s))) : smem_desc(rs_smem_addr(b_lo(s)));
        constexpr unsigned idesc = B_MN ? G::IDESC_BMN : G::IDESC;
#pragma unroll
        for (int k = 0; k < BK / 8; ++k) {
          // K-major: the next 8 K values are 32 bytes along the swizzled row;
          // MN-major: the next 8 K rows are the next 1 KiB atom
          const unsigned long long off = (unsigned long long)(k * 32) >> 4;
          const unsigned long long boff = B_MN ? (unsigned long long)(k * 1024) >> 4 : off;
          mma2(tmem, alo + off, bhi + boff, idesc, (kb != kb0 || k != 0) ? 1u : 0u);
          mma2(tmem, ahi + off, blo + boff, idesc, 1u);
          mma2(tmem, ahi + off, bhi + boff, idesc, 1u);
        }
        commit2_multicast(&empty[s]);
      }
      commit2_multicast(tmem_full);
    }
    __syncwarp();
  } else {
    const int t = threadIdx.x - 64;
    for (int kb = kb0; kb < kb1; ++kb) {
      const int s = (kb - kb0) % STAGES;
      const unsigned ph = (unsigned)(((kb - kb0) / STAGES) & 1);
      rs_mbar_wait(&full[s], ph);
      split_tile<false>(a_raw(s), a_lo(s), G::TILE_A, t);
      split_tile<false>(b_raw(s), b_lo(s), G::TILE_B, t);
      rs_fence_proxy_async();  // this thread's tile writes precede later async-proxy reads
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (t == 0) {
        if (rank == 0) {
          rs_mbar_arrive_expect_tx(&conv[s], 16u);  // the MMA issuer is in this CTA: CTA-scope release
        } else {
          signal_s2s_cluster(mapa(rs_smem_addr(sig_slot), 0u), sig_slot, mapa(rs_smem_addr(&conv[s]), 0u));
        }
      }
    }
    rs_mbar_wait(tmem_full, 0u);
    fence_after();
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const int trow = 128 * (int)rank + row;  // row within the 256-row pair tile
    const bool row_in = m0 + trow < M;
    float* crow = C + (long long)(row_in ? m0 + trow : 0) * ldc + n0;
    // columns [n0, n0 + ncols) exist; whole 16-byte groups when N % 4 == 0
    const int ncols = N - n0 < BN ? N - n0 : BN;
    auto store4 = [&](int col, float4 v) {  // col: tile column of v.x
      if (!row_in) return;
      if (N % 4 == 0 && col + 4 <= ncols) {
        *reinterpret_cast<float4*>(crow + col) = v;
      } else {
        if (col < ncols) crow[col] = v.x;
        if (col + 1 < ncols) crow[col + 1] = v.y;
        if (col + 2 < ncols) crow[col + 2] = v.z;
        if (col + 3 < ncols) crow[col + 3] = v.w;
      }
    };
    // split tiles: this CTA's half of the parked second-K-half tile and its flag
    float* wrow = ws + ((long long)(unit >> 1) * 256 + trow) * BN;
    unsigned* flag = flags + 2 * (unit >> 1) + rank;
    if (split && khalf == 0) {
      unsigned v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
      } while (v == 0u);
    }
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
      unsigned r[32];
      tmem_ld32(tmem + ((unsigned)(q * 32) << 16) + (unsigned)c0, r);
      if (!split) {
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          store4(c0 + j, make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]), __uint_as_float(r[j + 2]),
                                     __uint_as_float(r[j + 3])));
        }
      } else if (khalf == 1) {
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          __stcg(reinterpret_cast<float4*>(wrow + c0 + j),
                 make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]), __uint_as_float(r[j + 2]),
                             __uint_as_float(r[j + 3])));
        }
      } else {
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
          const float4 w = __ldcg(reinterpret_cast<const float4*>(wrow + c0 + j));
          store4(c0 + j,
                 make_float4(__fadd_rn(__uint_as_float(r[j]), w.x), __fadd_rn(__uint_as_float(r[j + 1]), w.y),
                             __fadd_rn(__uint_as_float(r[j + 2]), w.z), __fadd_rn(__uint_as_float(r[j + 3]), w.w)));
        }
      }
    }
    if (split) {
      // every epilogue thread of this CTA is done with the parked tile
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (t == 0) {
        if (khalf == 1) {
          asm volatile("fence.acq_rel.gpu;" ::: "memory");  // the parked tile before the flag
          asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flag), "r"(1u) : "memory");
        } else {
          *flag = 0u;  // consumed: ready for the next launch
        }
      }
    }
  }
  fence_before();
  cluster_sync();
  if (warp == 1) {
    fence_after();
    tmem_dealloc2<G::TMEM_COLS>(tmem);
  }
}

// Persistent form of gemm_3xtf32_2sm: one CTA pair per SM pair, looping over
// the same work units (whole tiles, then the K-split units) — unit u goes to
// pair u % P, so each pair owns at most one split unit, its last.  A split
// tile is cut into `ksplit` K ranges (2 for the tail past the last whole
// wave; up to 4 when the whole GEMM has fewer tiles than SM pairs, e.g. the
// 512-row A blocks of a strong-scaled multi-GPU sgemm): parts 1.. park their
// partial tiles in `ws` and count themselves into the tile's flag (release);
// part 0 waits for all of them (acquire) and stores
// C = ((part0 + part1) + part2) + ... — a fixed order, deterministic.
// The accumulator is double-buffered in TMEM (2 x BN columns): the MMA
// issuer fills slot i & 1 while four dedicated epilogue warps drain the
// other, so a tile's epilogue and the next tile's prologue overlap its
// neighbour's main loop.  Barriers: the stage ring (full / conv / empty) runs
// on a counter global to the pair's units; tmem_full[2] (MMA commit,
// multicast to both CTAs) and tmem_empty[2] (in CTA 0, one arrival per
// CTA's epilogue).  Warps: 0 TMA producer, 1 TMEM allocator + MMA issuer,
// 2..5 hi/lo converters, 6..9 epilogue (TMEM lane quarter = warp % 4).
constexpr int PTHREADS = 320;
constexpr int MAX_KSPLIT = 4;  // K parts per split tile (tmpl_gemm.schedule never exceeds it)

// Probe hook (tools/probe_gemm_timeline.py; compiled out unless the probe
// defines RS_GEMM_TIMELINE_OFFSET): %globaltimer of event e of the pair's
// i-th unit, recorded by CTA rank 0 past the end of the workspace.
#ifdef RS_GEMM_TIMELINE_OFFSET
#define RS_GEMM_TL(e, i)                                                                                   \
  do {                                                                                                     \
    if (rank == 0 && (i) < 16) {                                                                           \
      unsigned long long t_;                                                                               \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                              \
      reinterpret_cast<unsigned long long*>(ws + RS_GEMM_TIMELINE_OFFSET)[((long long)pair * 16 + (i)) * 8 + (e)] = t_; \
    }                                                                                                      \
  } while (0)
#else
#define RS_GEMM_TL(e, i) \
  do {                   \
  } while (0)
#endif

template <int M, int N, int K, int BN, int STAGES, bool B_MN = false, int GROUP_M = 0>
RS_DEVICE void gemm_3xtf32_2sm_persistent(float* __restrict__ C, int ldc, const rs_tmap* mapA, const rs_tmap* mapB,
                                          int n_full, int n_units, int ksplit, float* __restrict__ ws,
                                          unsigned* __restrict__ flags) {
  using G = Cfg2<BN, STAGES>;
  extern __shared__ __align__(1024) unsigned char rs_gemm_smem_raw[];
  unsigned char* smem =
      rs_gemm_smem_raw + ((1024u - (rs_smem_addr(rs_gemm_smem_raw) & 1023u)) & 1023u);
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem + STAGES * G::STAGE_BYTES);
  unsigned long long* full = bars;
  unsigned long long* conv = bars + STAGES;
  unsigned long long* empty = bars + 2 * STAGES;
  unsigned long long* tmem_full = bars + 3 * STAGES;       // [2]
  unsigned long long* tmem_empty = bars + 3 * STAGES + 2;  // [2]
  unsigned* tmem_slot = reinterpret_cast<unsigned*>(bars + 3 * STAGES + 4);
  unsigned char* sig_slot = reinterpret_cast<unsigned char*>(bars) + ((3 * STAGES + 5) * 8 + 15) / 16 * 16;

  constexpr int KB = (K + BK - 1) / BK;
  constexpr int NTN = (N + BN - 1) / BN;
  const unsigned rank = cluster_ctarank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  auto a_raw = [&](int s) { return smem + s * G::STAGE_BYTES; };
  auto a_lo = [&](int s) { return smem + s * G::STAGE_BYTES + G::TILE_A; };
  auto b_raw = [&](int s) { return smem + s * G::STAGE_BYTES + 2 * G::TILE_A; };
  auto b_lo = [&](int s) { return smem + s * G::STAGE_BYTES + 2 * G::TILE_A + G::TILE_B; };
  // unit -> (tile, K range, split part; sidx = the split tile's index or -1)
  auto unit_of = [&](int u, int& m0, int& n0, int& kb0, int& kb1, int& khalf, int& sidx) {
    const bool split = u >= n_full;
    const int su = split ? u - n_full : 0;
    sidx = split ? su / ksplit : -1;
    const int tile = split ? n_full + sidx : u;
    khalf = split ? su % ksplit : 0;
    kb0 = split ? (KB * khalf) / ksplit : 0;
    kb1 = split ? (KB * (khalf + 1)) / ksplit : KB;
    if (GROUP_M > 0) {  // tiles in groups of GROUP_M row tiles, column by column (L2 reuse of A and B)
      constexpr int NTM = (M + 255) / 256;
      const int grp = tile / (GROUP_M * NTN), r = tile % (GROUP_M * NTN);
      const int rows = NTM - grp * GROUP_M < GROUP_M ? NTM - grp * GROUP_M : GROUP_M;
      m0 = (grp * GROUP_M + r % rows) * 256;
      n0 = (r / rows) * BN;
    } else {
      m0 = (tile / NTN) * 256;
      n0 = (tile % NTN) * BN;
    }
  };

  if (threadIdx.x == 0) {
    if (ksplit > MAX_KSPLIT) __trap();  // the merge holds at most MAX_KSPLIT - 1 parked parts
    rs_tmap_prefetch(mapA);
    rs_tmap_prefetch(mapB);
    for (int s = 0; s < STAGES; ++s) {
      rs_mbar_init(&full[s], 1);
      rs_mbar_init(&conv[s], 1);
      rs_mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      rs_mbar_init(&tmem_full[a], 1);
      rs_mbar_init(&tmem_empty[a], 2);  // one arrival from each CTA's epilogue (CTA 0's copy is used)
    }
    rs_fence_barrier_init();
  }
  if (warp == 1) tmem_alloc2<2 * G::TMEM_COLS>(tmem_slot);
  fence_before();
  cluster_sync();
  fence_after();
  const unsigned tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int g = 0;
      for (int u = pair; u < n_units; u += npairs) {
        int m0, n0, kb0, kb1, khalf, sidx;
        unit_of(u, m0, n0, kb0, kb1, khalf, sidx);
        for (int kb = kb0; kb < kb1; ++kb, ++g) {
          const int s = g % STAGES;
          const unsigned ph = (unsigned)((g / STAGES) & 1);
          rs_mbar_wait(&empty[s], ph ^ 1u);
          rs_mbar_arrive_expect_tx(&full[s], G::TILE_A + G::TILE_B);
          rs_tma_load_2d(a_raw(s), mapA, kb * BK, m0 + 128 * (int)rank, &full[s]);
          if (B_MN) {
#pragma unroll
            for (int b = 0; b < BN / 64; ++b)
              rs_tma_load_2d(b_raw(s) + b * 4096, mapB, n0 + (BN / 2) * (int)rank + 32 * b, kb * BK, &full[s]);
          } else {
            rs_tma_load_2d(b_raw(s), mapB, kb * BK, n0 + (BN / 2) * (int)rank, &full[s]);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0 && lane == 0) {
      int g = 0, i = 0;
      constexpr unsigned idesc = B_MN ? G::IDESC_BMN : G::IDESC;
      for (int u = pair; u < n_units; u += npairs, ++i) {
        int m0, n0, kb0, kb1, khalf, sidx;
        unit_of(u, m0, n0, kb0, kb1, khalf, sidx);
        const int slot = i & 1;
        RS_GEMM_TL(0, i);
        if (i >= 2) mbar_wait_cluster(&tmem_empty[slot], (unsigned)(((i >> 1) & 1) ^ 1));
        fence_after();
        RS_GEMM_TL(1, i);
        const unsigned acc = tmem + (unsigned)(slot * BN);
        for (int kb = kb0; kb < kb1; ++kb, ++g) {
          const int s = g % STAGES;
          const unsigned ph = (unsigned)((g / STAGES) & 1);
          mbar_wait_cluster(&conv[s], ph);
          fence_after();
          if (kb == kb0) RS_GEMM_TL(2, i);
          const unsigned long long ahi = smem_desc(rs_smem_addr(a_raw(s)));
          const unsigned long long alo = smem_desc(rs_smem_addr(a_lo(s)));
          const unsigned long long bhi =
              B_MN ? smem_desc_mn(rs_smem_addr(b_raw(s))) : smem_desc(rs_smem_addr(b_raw(s)));
          const unsigned long long blo =
              B_MN ? smem_desc_mn(rs_smem_addr(b_lo(s))) : smem_desc(rs_smem_addr(b_lo(s)));
#pragma unroll
          for (int k = 0; k < BK / 8; ++k) {
            const unsigned long long off = (unsigned long long)(k * 32) >> 4;
            const unsigned long long boff = B_MN ? (unsigned long long)(k * 1024) >> 4 : off;
            mma2(acc, alo + off, bhi + boff, idesc, (kb != kb0 || k != 0) ? 1u : 0u);
            mma2(acc, ahi + off, blo + boff, idesc, 1u);
            mma2(acc, ahi + off, bhi + boff, idesc, 1u);
          }
          commit2_multicast(&empty[s]);
        }
        commit2_multicast(&tmem_full[slot]);
        RS_GEMM_TL(3, i);
      }
    }
    __syncwarp();
  } else if (warp < 6) {
    const int t = threadIdx.x - 64;
    int g = 0;
    for (int u = pair; u < n_units; u += npairs) {
      int m0, n0, kb0, kb1, khalf, sidx;
      unit_of(u, m0, n0, kb0, kb1, khalf, sidx);
      for (int kb = kb0; kb < kb1; ++kb, ++g) {
        const int s = g % STAGES;
        const unsigned ph = (unsigned)((g / STAGES) & 1);
        rs_mbar_wait(&full[s], ph);
        split_tile<false>(a_raw(s), a_lo(s), G::TILE_A, t);
        split_tile<false>(b_raw(s), b_lo(s), G::TILE_B, t);
        rs_fence_proxy_async();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (t == 0) {
          if (rank == 0) {
            rs_mbar_arrive_expect_tx(&conv[s], 16u);
          } else {
            signal_s2s_cluster(mapa(rs_smem_addr(sig_slot), 0u), sig_slot, mapa(rs_smem_addr(&conv[s]), 0u));
          }
        }
      }
    }
  } else {
    // epilogue warps 6..9
    const int t = threadIdx.x - 192;
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const int trow = 128 * (int)rank + row;
    int i = 0;
    for (int u = pair; u < n_units; u += npairs, ++i) {
      int m0, n0, kb0, kb1, khalf, sidx;
      unit_of(u, m0, n0, kb0, kb1, khalf, sidx);
      const bool split = sidx >= 0;
      const int slot = i & 1;
      rs_mbar_wait(&tmem_full[slot], (unsigned)((i >> 1) & 1));
      fence_after();
      if (t == 0) RS_GEMM_TL(4, i);
      const bool row_in = m0 + trow < M;
      float* crow = C + (long long)(row_in ? m0 + trow : 0) * ldc + n0;
      const int ncols = N - n0 < BN ? N - n0 : BN;
      auto store4 = [&](int col, float4 v) {
        if (!row_in) return;
        if (N % 4 == 0 && col + 4 <= ncols) {
          *reinterpret_cast<float4*>(crow + col) = v;
        } else {
          if (col < ncols) crow[col] = v.x;
          if (col + 1 < ncols) crow[col + 1] = v.y;
          if (col + 2 < ncols) crow[col + 2] = v.z;
          if (col + 3 < ncols) crow[col + 3] = v.w;
        }
      };
      const long long part_stride = 256LL * BN;
      if (split && ksplit == 2) {
        // Two K halves: each parks the column half the OTHER finalises (part 0
        // finalises columns [0, BN/2), part 1 [BN/2, BN)), signals, waits for the
        // other's, and adds the parked partial to its own: two half merges in
        // parallel instead of one whole-tile merge.  Same sum either way:
        // part0 + part1 (IEEE addition is commutative).  Flags: 4 per split tile
        // (part x CTA rank); each part resets the flag it consumed.
        const int own0 = khalf == 0 ? 0 : BN / 2, park0 = BN / 2 - own0;
        float* wtile = ws + (long long)sidx * part_stride + (long long)trow * BN;
        unsigned* myflag = flags + 4 * sidx + 2 * khalf + rank;
        unsigned* otherflag = flags + 4 * sidx + 2 * (1 - khalf) + rank;
#pragma unroll 1
        for (int c0 = park0; c0 < park0 + BN / 2; c0 += 32) {
          unsigned r[32];
          tmem_ld32(tmem + (unsigned)(slot * BN) + ((unsigned)(q * 32) << 16) + (unsigned)c0, r);
#pragma unroll
          for (int j = 0; j < 32; j += 4)
            __stcg(reinterpret_cast<float4*>(wtile + c0 + j),
                   make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]), __uint_as_float(r[j + 2]),
                               __uint_as_float(r[j + 3])));
        }
        asm volatile("bar.sync 2, 128;" ::: "memory");  // this CTA's half is parked
        if (t == 0) {
          asm volatile("fence.acq_rel.gpu;" ::: "memory");  // the parked half before the flag
          asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(myflag), "r"(1u) : "memory");
        }
        {
          unsigned v;
          do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(otherflag) : "memory");
          } while (v == 0u);
        }
        if (t == 0) RS_GEMM_TL(6, i);
#pragma unroll 1
        for (int c0 = own0; c0 < own0 + BN / 2; c0 += 32) {
          unsigned r[32];
          tmem_ld32(tmem + (unsigned)(slot * BN) + ((unsigned)(q * 32) << 16) + (unsigned)c0, r);
#pragma unroll
          for (int j = 0; j < 8; ++j) {  // (independent loads: the unrolled chunk issues them together)
            const float4 w = __ldcg(reinterpret_cast<const float4*>(wtile + c0 + 4 * j));
            store4(c0 + 4 * j, make_float4(__fadd_rn(__uint_as_float(r[4 * j]), w.x),
                                           __fadd_rn(__uint_as_float(r[4 * j + 1]), w.y),
                                           __fadd_rn(__uint_as_float(r[4 * j + 2]), w.z),
                                           __fadd_rn(__uint_as_float(r[4 * j + 3]), w.w)));
          }
        }
        fence_before();
        asm volatile("bar.sync 2, 128;" ::: "memory");
        if (t == 0) {
          *otherflag = 0u;  // consumed: ready for the next launch
          if (rank == 0) rs_mbar_arrive(&tmem_empty[slot]);
          else mbar_arrive_remote(mapa(rs_smem_addr(&tmem_empty[slot]), 0u));
          RS_GEMM_TL(5, i);
        }
        continue;
      }
      // parked parts of split tile sidx: part p (1 .. ksplit-1) at slot sidx * (ksplit-1) + p - 1
      float* wbase = ws + ((long long)(split ? sidx : 0) * (ksplit - 1)) * part_stride + (long long)trow * BN;
      float* wrow = wbase + (long long)(khalf > 0 ? khalf - 1 : 0) * part_stride;
      unsigned* flag = flags + 2 * (split ? sidx : 0) + rank;
      if (split && khalf == 0) {
        unsigned v;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
        } while (v < (unsigned)(ksplit - 1));
      }
      if (t == 0) RS_GEMM_TL(6, i);
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        unsigned r[32];
        tmem_ld32(tmem + (unsigned)(slot * BN) + ((unsigned)(q * 32) << 16) + (unsigned)c0, r);
        if (!split) {
#pragma unroll
          for (int j = 0; j < 32; j += 4)
            store4(c0 + j, make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]), __uint_as_float(r[j + 2]),
                                       __uint_as_float(r[j + 3])));
        } else if (khalf > 0) {
#pragma unroll
          for (int j = 0; j < 32; j += 4)
            __stcg(reinterpret_cast<float4*>(wrow + c0 + j),
                   make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]), __uint_as_float(r[j + 2]),
                               __uint_as_float(r[j + 3])));
        } else {
          // the parked parts of this 32-column chunk: every load issued before the
          // first add (one L2 round trip per chunk, not one per part and float4),
          // then the parts added in order: deterministic.  ksplit <= MAX_KSPLIT.
          float4 w[MAX_KSPLIT - 1][8];
#pragma unroll
          for (int p = 1; p < MAX_KSPLIT; ++p) {
            if (p < ksplit) {
#pragma unroll
              for (int j = 0; j < 8; ++j)
                w[p - 1][j] = __ldcg(reinterpret_cast<const float4*>(wbase + (long long)(p - 1) * part_stride + c0 + 4 * j));
            }
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            float4 a = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                   __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
#pragma unroll
            for (int p = 1; p < MAX_KSPLIT; ++p) {
              if (p < ksplit) {
                const float4 v = w[p - 1][j];
                a = make_float4(__fadd_rn(a.x, v.x), __fadd_rn(a.y, v.y), __fadd_rn(a.z, v.z), __fadd_rn(a.w, v.w));
              }
            }
            store4(c0 + 4 * j, a);
          }
        }
      }
      // this CTA's share of the slot is drained (and the parked tiles used)
      fence_before();
      asm volatile("bar.sync 2, 128;" ::: "memory");
      if (t == 0) {
        if (split && khalf > 0) {
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
          asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(flag), "r"(1u) : "memory");
        } else if (split) {
          *flag = 0u;
        }
        if (rank == 0) rs_mbar_arrive(&tmem_empty[slot]);
        else mbar_arrive_remote(mapa(rs_smem_addr(&tmem_empty[slot]), 0u));
        RS_GEMM_TL(5, i);
      }
    }
  }
  fence_before();
  cluster_sync();
  if (warp == 1) {
    fence_after();
    tmem_dealloc2<2 * G::TMEM_COLS>(tmem);
  }
}

}  // namespace rise_gemm
