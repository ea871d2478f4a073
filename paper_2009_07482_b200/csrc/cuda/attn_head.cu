// Fused attention-head chain for sm_100a (HS_OP_ATTN_HEAD):
//
//   Z[S, dW] = softmax_row(s · Q Kᵀ) · V · W        Q, K, V: [S, dk]  W: [dk, dW]
//
// which is the encoder head's ndrange chain gemm_nt(Q,K) -> softmax -> gemm(P,V)
// -> gemm(C,W_h) executed as one launch per batch of instances:
// the score matrix S, the probabilities P and the head output C never leave the
// SM (TMEM / shared memory), only Q, K, V are read and Z written.
//
// Persistent kernel, one CTA per SM walking instances. Per instance, all
// products are 3xTF32 on tcgen05 (A operand split hi/lo into TMEM, B split into
// shared memory; D += Alo·Bhi + Ahi·Blo + Ahi·Bhi in the same order as the
// unfused GEMM kernel, so each intermediate is bit-identical to what the
// unfused chain writes to HBM).
//
// Warp roles (512 threads):
//   warp 0      TMA: W planes once; per instance Q + K, then V into Q's buffer
//   warp 1      MMA issuer (one lane)
//   warp 2      TMEM allocator (512 columns)
//   warps 4-11  row warps: warp 4+q+4g owns TMEM lane quarter q (rows 32q..32q+31)
//               and column half g of every per-row pass: Q split -> TMEM; softmax
//               over the S accumulator (64 columns per thread held in registers,
//               row max / sum exchanged with the partner warp through smem) -> P
//               split -> TMEM; C (= P·V) split -> TMEM; Z -> TMA store. Two warps
//               per scheduler on the latency-bound row passes.
//   warps 12-15 operand warps: K -> tf32 hi (in place) / lo; V -> K-major hi / lo
//
// Softmax summation order: sequential over columns [0,64) and over [64,128), then
// s0 + s1 — the same order as the GEMM softmax epilogue (gemm_tc.cu), so the fused
// head stays bit-identical to the unfused chain.
//
// TMEM columns: [0,128) S accumulator | [128,384) A operand region: Q hi/lo,
// then P hi/lo, then C hi/lo | [384,448) C accumulator | [448,512) Z accumulator.
#include <mutex>

#include "kernels.cuh"
#include "launch.cuh"
#include "tc_common.cuh"

namespace hs {

namespace {

using namespace tc;

constexpr int kS = 128;  // max rows = keys per head (one M tile; softmax width <= 128)
constexpr int kDK = 64;  // head width: K of QKᵀ, N of P·V, K of C·W
constexpr int kDW = 64;  // output width: N of C·W
constexpr int kAttnThreads = 512;

// shared memory regions (bytes from the 1024-aligned base)
constexpr uint32_t kQV = 0;                  // Q staging: 2 SW128 tiles [128 rows][32 k] (32 KB); then V staging
constexpr uint32_t kKhi = kQV + 32768;       // K staging [128 n][32 k] x 2, converted to tf32 hi in place
constexpr uint32_t kKlo = kKhi + 32768;      // K lo
constexpr uint32_t kVop = kKlo + 32768;      // V operand: hi 4 x [64 n][32 k] SW128 (32 KB), lo (32 KB)
constexpr uint32_t kW = kVop + 65536;        // W planes: hi 2 x [64 n][32 k] (16 KB), lo (16 KB)
constexpr uint32_t kEpi = kW + 32768;        // Z staging: 8 warps x [32 rows][32 cols] (32 KB); its first
                                             // 256 B per warp also carry the softmax row max / sum exchange
constexpr uint32_t kBar = kEpi + 32768;      // mbarriers + TMEM slot
constexpr int kAttnSmem = int(kBar) + 256 + 1024;

enum Bar : uint32_t {
  QK_FULL, V_FULL, W_FULL, Q_FREE, K_READY, A_READY, S_FULL, P_READY, VB_READY, V_FREE, O_FULL, C_READY, Z_FULL,
  TMEM_SLOT
};

struct AttnParams {
  int S;      // rows = keys (<= 128)
  int batch;
  float scale;
};

// split 16 fp32 -> tf32 hi / lo registers
__device__ __forceinline__ void split16(const float (&x)[16], uint32_t (&hi)[16], uint32_t (&lo)[16]) {
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const float h = tf32_rna(x[e]);
    hi[e] = __float_as_uint(h);
    lo[e] = __float_as_uint(tf32_lo(x[e], h));
  }
}

template <int kTerms>
__device__ __forceinline__ void mma3(uint32_t d, uint32_t a_hi, uint32_t a_lo, uint32_t b_hi, uint32_t b_lo,
                                     uint32_t idesc, uint32_t first) {
  if constexpr (kTerms > 1) {
    mma_tf32_ts(d, a_lo, smem_desc(b_hi), idesc, first);
    mma_tf32_ts(d, a_hi, smem_desc(b_lo), idesc, 1u);
    mma_tf32_ts(d, a_hi, smem_desc(b_hi), idesc, 1u);
  } else {
    mma_tf32_ts(d, a_hi, smem_desc(b_hi), idesc, first);
  }
}

template <int kTerms>
__global__ void __launch_bounds__(kAttnThreads, 1)
    attn_head_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmW,
                     const __grid_constant__ CUtensorMap tmZ, AttnParams p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  auto bar = [&](uint32_t b) { return base + kBar + 8u * b; };
  const uint32_t* tmem_slot_ptr =
      reinterpret_cast<const uint32_t*>(smem_raw + (bar(TMEM_SLOT) - smem_u32(smem_raw)));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    mbar_init(bar(QK_FULL), 1);
    mbar_init(bar(V_FULL), 1);
    mbar_init(bar(W_FULL), 1);
    for (uint32_t b : {Q_FREE, A_READY, P_READY, C_READY}) mbar_init(bar(b), 8);  // row warps
    for (uint32_t b : {K_READY, VB_READY, V_FREE}) mbar_init(bar(b), 4);           // operand warps
    for (uint32_t b : {S_FULL, O_FULL, Z_FULL}) mbar_init(bar(b), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (const CUtensorMap* m : {&tmQ, &tmK, &tmV, &tmW, &tmZ})
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(bar(TMEM_SLOT)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_launch_dependents();  // PDL (launch.cuh)
  pdl_wait();
  const uint32_t tmem = *tmem_slot_ptr;
  constexpr uint32_t kTS = 0, kTA = 128, kTC = 384, kTZ = 448;  // TMEM column offsets

  if (warp == 0) {
    // -------------------------------------------------------------- TMA producer
    if (lane == 0) {
      mbar_expect_tx(bar(W_FULL), 32768);
      for (int pl = 0; pl < 2; ++pl)
        for (int kb = 0; kb < 2; ++kb)
          tma_load_3d(base + kW + uint32_t(pl) * 16384u + uint32_t(kb) * 8192u, &tmW, bar(W_FULL), kb * BK, 0, pl);
      uint32_t i = 0;
      for (int inst = blockIdx.x; inst < p.batch; inst += gridDim.x, ++i) {
        if (i > 0) {
          mbar_wait(bar(V_FREE), (i - 1) & 1u);  // Q/V staging free (V of i-1 converted)
          mbar_wait(bar(S_FULL), (i - 1) & 1u);  // K operand free (QKᵀ of i-1 done)
        }
        mbar_expect_tx(bar(QK_FULL), 65536);
        for (int kb = 0; kb < 2; ++kb) {
          tma_load_3d(base + kQV + uint32_t(kb) * 16384u, &tmQ, bar(QK_FULL), kb * BK, 0, inst);
          tma_load_3d(base + kKhi + uint32_t(kb) * 16384u, &tmK, bar(QK_FULL), kb * BK, 0, inst);
        }
        mbar_wait(bar(Q_FREE), i & 1u);  // Q consumed by the row warps
        mbar_expect_tx(bar(V_FULL), 32768);
        for (int kb = 0; kb < 4; ++kb)
          tma_load_3d(base + kQV + uint32_t(kb) * 8192u, &tmV, bar(V_FULL), 0, kb * BK, inst);
      }
    }
  } else if (warp == 1) {
    // -------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idS = instr_desc_tf32(kS), id64 = instr_desc_tf32(kDK);
      mbar_wait(bar(W_FULL), 0);
      uint32_t i = 0;
      for (int inst = blockIdx.x; inst < p.batch; inst += gridDim.x, ++i) {
        const uint32_t ph = i & 1u;
        // S = Q Kᵀ (K = dk = 64)
        mbar_wait(bar(A_READY), ph);
        mbar_wait(bar(K_READY), ph);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < kDK / 8; ++kk) {
          const uint32_t kbo = uint32_t(kk >> 2) * 16384u + uint32_t(kk & 3) * 32u;
          mma3<kTerms>(tmem + kTS, tmem + kTA + uint32_t(kk) * 8u, tmem + kTA + 64u + uint32_t(kk) * 8u,
                       base + kKhi + kbo, base + kKlo + kbo, idS, kk ? 1u : 0u);
        }
        mma_commit(bar(S_FULL));
        // C = P V (K = S keys = 128)
        mbar_wait(bar(P_READY), ph);
        mbar_wait(bar(VB_READY), ph);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < kS / 8; ++kk) {
          const uint32_t kbo = uint32_t(kk >> 2) * 8192u + uint32_t(kk & 3) * 32u;
          mma3<kTerms>(tmem + kTC, tmem + kTA + uint32_t(kk) * 8u, tmem + kTA + 128u + uint32_t(kk) * 8u,
                       base + kVop + kbo, base + kVop + 32768u + kbo, id64, kk ? 1u : 0u);
        }
        mma_commit(bar(O_FULL));
        // Z = C W (K = dk = 64)
        mbar_wait(bar(C_READY), ph);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < kDK / 8; ++kk) {
          const uint32_t kbo = uint32_t(kk >> 2) * 8192u + uint32_t(kk & 3) * 32u;
          mma3<kTerms>(tmem + kTZ, tmem + kTA + uint32_t(kk) * 8u, tmem + kTA + 64u + uint32_t(kk) * 8u,
                       base + kW + kbo, base + kW + 16384u + kbo, id64, kk ? 1u : 0u);
        }
        mma_commit(bar(Z_FULL));
      }
    }
  } else if (warp >= 4 && warp < 12) {
    // -------------------------------------------------------------- row warps
    const int q = warp & 3, g = (warp - 4) >> 2, row = q * 32 + lane;
    const uint32_t lane_base = tmem + (uint32_t(q * 32) << 16);
    const uint32_t stage = base + kEpi + uint32_t(q * 2 + g) * 4096u;
    // softmax exchange with the partner warp (same lane quarter, other column half):
    // max at stage[lane], sum at stage[32 + lane] of each warp's own staging tile
    const uint32_t mine = stage + uint32_t(lane) * 4u;
    const uint32_t other = base + kEpi + uint32_t(q * 2 + (g ^ 1)) * 4096u + uint32_t(lane) * 4u;
    const float sl = p.scale * 1.4426950408889634f;
    uint32_t i = 0;
    for (int inst = blockIdx.x; inst < p.batch; inst += gridDim.x, ++i) {
      const uint32_t ph = i & 1u;
      // (A) Q row, columns [32g, 32g+32) -> tf32 hi [kTA, kTA+64) / lo [kTA+64, kTA+128)
      mbar_wait(bar(QK_FULL), ph);
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        float x[16];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float4 v = lds128(base + kQV + uint32_t(g) * 16384u + sw128(row, 4 * hh + c));
          x[4 * c] = v.x; x[4 * c + 1] = v.y; x[4 * c + 2] = v.z; x[4 * c + 3] = v.w;
        }
        uint32_t hi[16], lo[16];
        split16(x, hi, lo);
        const uint32_t col = kTA + uint32_t(g * 32 + hh * 16);
        tmem_st16(lane_base + col, hi);
        tmem_st16(lane_base + col + 64u, lo);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(bar(A_READY));
        mbar_arrive(bar(Q_FREE));
      }
      // (B) softmax over S columns [64g, 64g+64) held in registers -> P hi [kTA, kTA+128) / lo [+128)
      mbar_wait(bar(S_FULL), ph);
      tc_fence_after();
      uint32_t r0[32], r1[32];
      tmem_ld32_nowait(lane_base + kTS + uint32_t(g * 64), r0);
      tmem_ld32_nowait(lane_base + kTS + uint32_t(g * 64 + 32), r1);
      tmem_ld_wait(r0);
      tmem_ld_dep(r1);
      // S is consumed (registers): nothing else of this instance reads it
      float mx = -INFINITY;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if (g * 64 + j < p.S) mx = fmaxf(mx, __uint_as_float(r0[j]) * p.scale);
        if (g * 64 + 32 + j < p.S) mx = fmaxf(mx, __uint_as_float(r1[j]) * p.scale);
      }
      if (i > 0) {  // the previous Z store has finished reading this warp's staging tile
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncwarp();
      }
      sts32(mine, mx);
      named_bar(1u + uint32_t(q), 64u);  // the two warps of lane quarter q
      mx = fmaxf(mx, lds32(other));
      const float ml = mx * 1.4426950408889634f;
      float sum = 0.f;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float e = g * 64 + j < p.S ? ex2_approx(fmaf(__uint_as_float(r0[j]), sl, -ml)) : 0.f;
        sum = sum + e;
        r0[j] = __float_as_uint(e);
      }
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float e = g * 64 + 32 + j < p.S ? ex2_approx(fmaf(__uint_as_float(r1[j]), sl, -ml)) : 0.f;
        sum = sum + e;
        r1[j] = __float_as_uint(e);
      }
      sts32(mine + 128u, sum);
      named_bar(1u + uint32_t(q), 64u);
      const float s_other = lds32(other + 128u);
      const float inv = 1.f / (g == 0 ? sum + s_other : s_other + sum);  // s0 + s1
      // P = e * inv split in place: r -> hi (tmem_st16 reads it), lo computed alongside
#pragma unroll
      for (int hh = 0; hh < 4; ++hh) {
        uint32_t hi[16], lo[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const float x = __uint_as_float(hh < 2 ? r0[(hh & 1) * 16 + e] : r1[(hh & 1) * 16 + e]) * inv;
          const float h = tf32_rna(x);
          hi[e] = __float_as_uint(h);
          lo[e] = __float_as_uint(tf32_lo(x, h));
        }
        const uint32_t col = kTA + uint32_t(g * 64 + hh * 16);
        tmem_st16(lane_base + col, hi);
        tmem_st16(lane_base + col + 128u, lo);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar(P_READY));
      // (C) C = P·V accumulator columns [32g, 32g+32) -> tf32 hi [kTA, kTA+64) / lo [kTA+64, kTA+128)
      mbar_wait(bar(O_FULL), ph);
      tc_fence_after();
      {
        uint32_t r[32];
        tmem_ld32(lane_base + kTC + uint32_t(g * 32), r);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          float x[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) x[e] = __uint_as_float(r[hh * 16 + e]);
          uint32_t hi[16], lo[16];
          split16(x, hi, lo);
          const uint32_t col = kTA + uint32_t(g * 32 + hh * 16);
          tmem_st16(lane_base + col, hi);
          tmem_st16(lane_base + col + 64u, lo);
        }
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar(C_READY));
      // (D) Z accumulator columns [32g, 32g+32) -> SW128 staging -> TMA store (rows >= S clipped by the map)
      mbar_wait(bar(Z_FULL), ph);
      tc_fence_after();
      {
        uint32_t r[32];
        tmem_ld32(lane_base + kTZ + uint32_t(g * 32), r);  // the partner read this tile's exchange
                                                              // words before arriving on P_READY
#pragma unroll
        for (int c = 0; c < 8; ++c)
          sts128(stage + uint32_t(lane) * 128u + (uint32_t(c ^ (lane & 7)) << 4),
                 make_float4(__uint_as_float(r[4 * c]), __uint_as_float(r[4 * c + 1]), __uint_as_float(r[4 * c + 2]),
                             __uint_as_float(r[4 * c + 3])));
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) tma_store_3d(&tmZ, stage, g * 32, q * 32, inst);
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  } else if (warp >= 12) {
    // -------------------------------------------------------------- operand warps
    const int t = threadIdx.x - 384;  // 0..127
    uint32_t i = 0;
    for (int inst = blockIdx.x; inst < p.batch; inst += gridDim.x, ++i) {
      const uint32_t ph = i & 1u;
      // K [n][k] SW128 staging -> hi in place, lo alongside (same offsets)
      mbar_wait(bar(QK_FULL), ph);
#pragma unroll 4
      for (int j = 0; j < 16; ++j) {
        const uint32_t off = uint32_t(t + 128 * j) * 16u;
        const float4 x = lds128(base + kKhi + off);
        const float4 h = make_float4(tf32_rna(x.x), tf32_rna(x.y), tf32_rna(x.z), tf32_rna(x.w));
        sts128(base + kKhi + off, h);
        sts128(base + kKlo + off, tf32_lo4(x, h));
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(bar(K_READY));
      // V [32 k][64 n] staging (x4) -> K-major SW128 hi/lo tiles [64 n][32 k] (x4)
      mbar_wait(bar(V_FULL), ph);
      if (i > 0) mbar_wait(bar(O_FULL), (i - 1) & 1u);  // P·V of i-1 has read the V operand
#pragma unroll 2
      for (int j = 0; j < 16; ++j) {
        const int id = t + 128 * j;  // 4 k-blocks x 64 n x 8 chunks of 4 k
        const int kb = id >> 9, n = id & 63, kc = (id >> 6) & 7;
        const uint32_t src = base + kQV + uint32_t(kb) * 8192u + uint32_t((kc * 4) * 64 + n) * 4u;
        const float4 x = make_float4(lds32(src), lds32(src + 256), lds32(src + 512), lds32(src + 768));
        const float4 h = make_float4(tf32_rna(x.x), tf32_rna(x.y), tf32_rna(x.z), tf32_rna(x.w));
        const uint32_t dst = base + kVop + uint32_t(kb) * 8192u + sw128(n, kc);
        sts128(dst, h);
        sts128(dst + 32768u, tf32_lo4(x, h));
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(bar(VB_READY));
        mbar_arrive(bar(V_FREE));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

}  // namespace

bool attn_head_supported(const AttnArgs& a) {
  if (a.S < 1 || a.S > kS || a.dk != kDK || a.dw != kDW || a.batch < 1 || !a.Wplanes) return false;
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  if (!al16(a.Q) || !al16(a.K) || !al16(a.V) || !al16(a.Z) || !al16(a.Wplanes)) return false;
  const int64_t ld = a.ldz ? a.ldz : kDW;
  if ((a.sQ | a.sK | a.sV | a.sZ | ld) & 3) return false;
  return encode_fn() != nullptr;
}

cudaError_t attn_head(const AttnArgs& a, int terms, cudaStream_t s) {
  if (!attn_head_supported(a)) return cudaErrorInvalidValue;
  auto kernel = terms > 1 ? attn_head_kernel<3> : attn_head_kernel<1>;
  static std::once_flag once3, once1;
  static cudaError_t err3 = cudaSuccess, err1 = cudaSuccess;
  std::call_once(terms > 1 ? once3 : once1, [&] {
    (terms > 1 ? err3 : err1) = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kAttnSmem);
  });
  if (cudaError_t e = terms > 1 ? err3 : err1) return e;
  const uint64_t S = uint64_t(a.S), B = uint64_t(a.batch);
  const uint64_t ldz = uint64_t(a.ldz ? a.ldz : kDW);
  CUtensorMap mQ, mK, mV, mW, mZ;
  bool ok = make_map(&mQ, a.Q, kDK, S, B, kDK * 4, uint64_t(a.sQ ? a.sQ : S * kDK) * 4, BK, kS, true) &&
            make_map(&mK, a.K, kDK, S, B, kDK * 4, uint64_t(a.sK ? a.sK : S * kDK) * 4, BK, kS, true) &&
            make_map(&mV, a.V, kDK, S, B, kDK * 4, uint64_t(a.sV ? a.sV : S * kDK) * 4, kDK, BK, false) &&
            make_map(&mW, a.Wplanes, kDK, kDW, 2, kDK * 4, uint64_t(kDK * kDW) * 4, BK, kDW, true) &&
            make_map(&mZ, a.Z, kDW, S, B, ldz * 4, uint64_t(a.sZ ? a.sZ : S * ldz) * 4, 32, 32, true);
  if (!ok) return cudaErrorInvalidValue;
  AttnParams p{a.S, a.batch, a.scale};
  const int grid = a.batch < num_sms() ? a.batch : num_sms();
  return launch_node(kernel, dim3(grid), dim3(kAttnThreads), kAttnSmem, s, 1, mQ, mK, mV, mW, mZ, p);
}

}  // namespace hs
