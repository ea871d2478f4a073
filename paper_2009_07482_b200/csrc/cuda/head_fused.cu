// Whole transformer head as one sm_100a launch (HS_OP_HEAD):
//
//   Q | K | V = X · [Wq | Wk | Wv]         X: [S, D]   W*: [D, 64]   (resident, pre-split)
//   Z         = softmax_row(s · Q Kᵀ) · V · Wh              Wh: [64, 64] (resident, pre-split)
//
// which is the head component of the encoder DAG (SURVEY.md §8 C3:
// three projection GEMMs, transpose, QKᵀ, softmax, P·V, C·W_h) after the engine's
// launch rewrites: the grouped Q/K/V projection (gemm_tc.cu, gemm_pair_kernel<192>)
// and the fused attention chain (attn_head.cu) in one kernel, so Q, K, V never
// leave the SM. Each product is 3xTF32 with the operand split and the MMA order of
// those two kernels.
//
// CTA pair (cluster of 2 on one TPC) per pair of instances, persistent over pairs.
// Phase 1 (projection): the pair GEMM main loop with M = 256 (each CTA its own
// instance's 128 rows), N = 192, K = D: X tiles by TMA into staging, split hi/lo
// into TMEM by the converter warps, W planes by TMA (each CTA half of N).
// Phase 2 (attention), all MMAs still cta_group::2 with M = 256:
//   S  = [Q0;Q1] [K0;K1]ᵀ   N = 256: B rows 0-127 are CTA 0's keys, 128-255 CTA 1's;
//                           CTA r keeps its own block, columns [128r, 128r+128)
//   C  = [P0;P1] [V0 V1]    N = 128: B = Vᵀ, rows 0-63 CTA 0's, 64-127 CTA 1's;
//                           CTA r keeps columns [64r, 64r+64)
//   Z  = [C0;C1] Wh         N = 64: each CTA holds half of Whᵀ's rows
// The off-diagonal blocks of S and C are computed and discarded (2x the QKᵀ and
// P·V flops, 14 % of the head's): the price of one cta_group for the whole kernel.
//
// Warp roles (512 threads):
//   warp 0      TMA: X tiles (phase 1)
//   warp 1      MMA issuer (leader CTA, one lane)
//   warp 2      TMEM allocator (512 columns, cta_group::2)
//   warp 3      TMA: W planes (phase 1, this CTA's half of N), Wh half once
//   warps 4-11  phase 1: converters, group g = (w-4)/4 takes every other K-block
//               phase 2: row warps, TMEM lane quarter q = w%4, column half g:
//               Q split -> TMEM; softmax (S in registers, row max / sum exchanged
//               with the partner warp); C split -> TMEM; Z -> TMA store
//   warps 12-15 phase 2: K -> K-major smem hi/lo; V -> Vᵀ K-major smem hi/lo
//
// TMEM columns: phase 1: QKV accumulator [0,192) | A stages [192,448).
// phase 2: S [0,256) -> C acc [0,128) + Z acc [128,192); A operand [256,512):
// Q hi/lo [256,384) -> P hi/lo [256,512) -> C hi/lo [256,384).
#include <mutex>

#include "kernels.cuh"
#include "tc_common.cuh"

#ifndef HS_DBG_TIMELINE
#define HS_DBG_TIMELINE 0
#endif
#ifndef HS_DBG_HEAD_NOCONV  // timing experiment only (wrong results): skip the X split in phase 1
#define HS_DBG_HEAD_NOCONV 0
#endif

namespace hs {

#if HS_DBG_TIMELINE
// timing experiment only (profiles/head_timeline.py): clock64 stamps of cluster 0,
// CTA 0, first 8 pairs x 16 points
__device__ long long g_head_timeline[8 * 16];
#define TL(t, k)                                                             \
  do {                                                                       \
    if (pair0 == 0 && rank == 0 && (t) < 8) g_head_timeline[(t) * 16 + (k)] = clock64(); \
  } while (0)
#else
#define TL(t, k) \
  do {           \
  } while (0)
#endif

namespace {

using namespace tc;

constexpr int kS = 128, kDK = 64, kN = 3 * kDK;  // rows, head width, projection width
constexpr int kThreads = 512;
// Variant (measured slower, kept for A/B): three converter groups (warps 12-15
// convert too) with 6 X / 3 W+A stages. The projection drops from ~21k to ~19.6k
// cycles per pair, but stage 0 can be pre-converted for only a third of the
// pairs, and the first K-blocks of a pair wait for O_FULL: 105 vs 99 us per
// 512-instance launch (profiles/README.md).
#ifndef HS_HEAD_CONV3
#define HS_HEAD_CONV3 0
#endif
constexpr int kConv = HS_HEAD_CONV3 ? 3 : 2;  // converter groups (each takes every kConv-th K-block)
constexpr int kNS = HS_HEAD_CONV3 ? 6 : 4;    // X staging stages
constexpr int kNO = HS_HEAD_CONV3 ? 3 : 4;    // W operand stages = TMEM A stages
constexpr uint32_t kStaging = BM * BK * 4;            // 16 KB X tile
constexpr uint32_t kPlaneB = (kN / 2) * 128;          // 96 rows x 128 B: this CTA's half of N
constexpr uint32_t kOperand = 2 * kPlaneB;            // hi + lo
// shared memory (bytes from the 1024-aligned base)
constexpr uint32_t kU = 0;                            // union: phase 1 stages | phase 2 operands
constexpr uint32_t kOpB = kU + kNS * kStaging;        // phase 1 W operand ring
constexpr uint32_t kKop = kU;                         // phase 2: K hi/lo, 2 planes x 2 k-blocks x [128][128 B]
constexpr uint32_t kVop = kU + 65536;                 // phase 2: Vᵀ hi/lo, 2 planes x 4 k-blocks x [64][128 B]
constexpr uint32_t kUEnd = kOpB + kNO * kOperand;     // 160 KB
constexpr uint32_t kWh = kUEnd;                       // Whᵀ half: 2 planes x 2 k-blocks x [32][128 B] (16 KB)
constexpr uint32_t kEpi = kWh + 16384;                // Z staging: 4 warps x 2 x [32][32] fp32 (32 KB)
constexpr uint32_t kExch = kEpi + 32768;              // softmax row max / sum exchange: 8 warps x 2 x 32 fp32
constexpr uint32_t kBar = kExch + 2048;
constexpr int kSmem = int(kBar) + 512 + 1024;
static_assert(kVop + 65536 <= kUEnd, "phase 2 operands exceed the union");
static_assert(kSmem <= 227 * 1024, "shared memory budget exceeded");

constexpr uint32_t kTQ = 256;  // TMEM A-operand region (phase 2)
constexpr uint32_t kTZ = 448;  // Z accumulator: P lo's columns, free after P·V; outside the projection's TMEM
constexpr uint32_t kTStage = 192;

enum Bar : uint32_t {
  ST_FULL = 0,             // [kNS] local
  ST_EMPTY = ST_FULL + kNS,  // [kNS] local, 4 converter warps
  OP_FULL = ST_EMPTY + kNS,  // [kNO] leader: 2 x 4 converter warps + expect_tx
  OP_EMPTY = OP_FULL + kNO,  // [kNO] each CTA (commit multicast)
  ACC_FULL = OP_EMPTY + kNO,
  A_READY,   // leader: Q split + K operand, 2 x 8 warps (S = Q Kᵀ may start)
  V_READY,   // leader: Vᵀ operand, 2 x 8 warps (P·V may start)
  S_FULL,    // each CTA
  P_READY,   // leader: 2 x 8
  O_FULL,    // each CTA
  C_READY,   // leader: 2 x 8
  Z_FULL,    // each CTA
  WH_FULL,   // leader: expect_tx
  TMEM_SLOT,
  kNumBars
};
static_assert(kNumBars * 8 <= 512, "barrier area");

struct HeadParams {
  int S, D, batch, pairs;
  float scale;
};

template <int kTerms>
__device__ __forceinline__ void mma3(uint32_t d, uint32_t a_hi, uint32_t a_lo, uint32_t b_hi, uint32_t b_lo,
                                     uint32_t idesc, uint32_t first) {
  if constexpr (kTerms > 1) {
    mma_pair_tf32_ts(d, a_lo, smem_desc(b_hi), idesc, first);
    mma_pair_tf32_ts(d, a_hi, smem_desc(b_lo), idesc, 1u);
    mma_pair_tf32_ts(d, a_hi, smem_desc(b_hi), idesc, 1u);
  } else {
    mma_pair_tf32_ts(d, a_hi, smem_desc(b_hi), idesc, first);
  }
}

template <int kTerms>
__device__ __forceinline__ void split_row16(const uint32_t* r, uint32_t (&hi)[16], uint32_t (&lo)[16]) {
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const float x = __uint_as_float(r[e]);
    const float h = tf32_rna(x);
    hi[e] = __float_as_uint(h);
    lo[e] = __float_as_uint(x - h);
  }
}

// Softmax passes over this thread's 64 S values (columns c0.. of its row): the
// max of x·scale over valid keys, then e = 2^(x·scale·log2e - max·log2e) in place
// with their sequential sum (columns >= S give e = 0 when kMask).
template <bool kMask>
__device__ __forceinline__ float row_max(const uint32_t (&r0)[32], const uint32_t (&r1)[32], int c0, int S,
                                         float scale) {
  float mx = -INFINITY;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    if (!kMask || c0 + j < S) mx = fmaxf(mx, __uint_as_float(r0[j]) * scale);
    if (!kMask || c0 + 32 + j < S) mx = fmaxf(mx, __uint_as_float(r1[j]) * scale);
  }
  return mx;
}
template <bool kMask>
__device__ __forceinline__ float row_exp(uint32_t (&r0)[32], uint32_t (&r1)[32], int c0, int S, float sl, float ml) {
  float sum = 0.f;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const float e = (!kMask || c0 + j < S) ? ex2_approx(fmaf(__uint_as_float(r0[j]), sl, -ml)) : 0.f;
    sum = sum + e;
    r0[j] = __float_as_uint(e);
  }
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const float e = (!kMask || c0 + 32 + j < S) ? ex2_approx(fmaf(__uint_as_float(r1[j]), sl, -ml)) : 0.f;
    sum = sum + e;
    r1[j] = __float_as_uint(e);
  }
  return sum;
}

// K row (this key = TMEM lane) -> K-major SW128 tiles [128 keys][32 d] x 2 (hi at +0, lo at +32 KB)
__device__ __forceinline__ void store_k_operand(uint32_t base, uint32_t lane_base, int key) {
#pragma unroll 1
  for (int kb = 0; kb < 2; ++kb) {
    uint32_t r[32];
    tmem_ld32(lane_base + uint32_t(kDK + kb * 32), r);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const float4 x = make_float4(__uint_as_float(r[4 * c]), __uint_as_float(r[4 * c + 1]),
                                   __uint_as_float(r[4 * c + 2]), __uint_as_float(r[4 * c + 3]));
      const float4 h = make_float4(tf32_rna(x.x), tf32_rna(x.y), tf32_rna(x.z), tf32_rna(x.w));
      const uint32_t dst = base + kKop + uint32_t(kb) * 16384u + sw128(key, c);
      sts128(dst, h);
      sts128(dst + 32768u, make_float4(x.x - h.x, x.y - h.y, x.z - h.z, x.w - h.w));
    }
  }
}

// V row (this key = TMEM lane q*32 + lane), d in [32 half, 32 half + 32) -> Vᵀ K-major
// SW128 tiles [64 d][32 keys] (k-block = key / 32 = q; hi at +0, lo at +32 KB)
__device__ __forceinline__ void store_vt_operand(uint32_t base, uint32_t lane_base, int q, int lane, int half) {
  uint32_t r[32];
  tmem_ld32(lane_base + uint32_t(2 * kDK + half * 32), r);
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const int n = half * 32 + j;
    const float x = __uint_as_float(r[j]);
    const float h = tf32_rna(x);
    const uint32_t dst = base + kVop + uint32_t(q) * 8192u + sw128(n, lane >> 2) + uint32_t(lane & 3) * 4u;
    sts32(dst, h);
    sts32(dst + 32768u, x - h);
  }
}

template <int kTerms>
__global__ void __launch_bounds__(kThreads, 1)
    head_pair_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                     const __grid_constant__ CUtensorMap tmWh, const __grid_constant__ CUtensorMap tmZ, HeadParams p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  auto bar = [&](uint32_t b) { return base + kBar + 8u * b; };
  const uint32_t* tmem_slot_ptr =
      reinterpret_cast<const uint32_t*>(smem_raw + (bar(TMEM_SLOT) - smem_u32(smem_raw)));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int pair0 = int(cluster_id_x()), npairs = int(nclusters_x());
  const int nk = p.D / BK;
  auto leader = [&](uint32_t b) { return mapa_rank(bar(b), 0); };

  if (threadIdx.x == 0) {
    for (int s = 0; s < kNS; ++s) {
      mbar_init(bar(ST_FULL + s), 1);
      mbar_init(bar(ST_EMPTY + s), 4);
    }
    for (int o = 0; o < kNO; ++o) {
      mbar_init(bar(OP_FULL + o), 2 * 4 + 1);
      mbar_init(bar(OP_EMPTY + o), 1);
    }
    for (uint32_t b : {ACC_FULL, S_FULL, O_FULL, Z_FULL, WH_FULL}) mbar_init(bar(b), 1);
    mbar_init(bar(A_READY), 2 * 8);
    mbar_init(bar(V_READY), 2 * 8);
    for (uint32_t b : {P_READY, C_READY}) mbar_init(bar(b), 2 * 8);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (const CUtensorMap* m : {&tmX, &tmW, &tmWh, &tmZ})
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(bar(TMEM_SLOT)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot_ptr;

  if (warp == 0) {
    // ------------------------------------------------------------ X producer
    if (lane == 0) {
      uint32_t it = 0, lt = 0;
      for (int t = pair0; t < p.pairs; t += npairs, ++lt) {
        // X stages share the K operand's smem: free once the last pair's S = Q Kᵀ is done
        if (lt > 0) mbar_wait(bar(S_FULL), (lt - 1) & 1u);
        const int inst = 2 * t + int(rank);  // >= batch: zero-filled box
        bool o_waited = lt == 0;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = int(it % kNS);
          if (s >= 4 && !o_waited) {  // stages 4-5 share the Vᵀ operand's smem: wait for P·V
            mbar_wait(bar(O_FULL), (lt - 1) & 1u);
            o_waited = true;
          }
          mbar_wait(bar(ST_EMPTY + s), ((it / kNS) & 1u) ^ 1u);
          mbar_expect_tx(bar(ST_FULL + s), kStaging);
          tma_load_3d(base + kU + uint32_t(s) * kStaging, &tmX, bar(ST_FULL + s), kb * BK, 0, inst);
        }
        // warm L2 with this CTA's rows of the next pair: its loads start only after
        // phase 2, and would otherwise pay the HBM latency at the head of the pipeline
        if (t + npairs < p.pairs)
          for (int kb = 0; kb < nk; ++kb) tma_prefetch_3d(&tmX, kb * BK, 0, 2 * (t + npairs) + int(rank));
      }
    }
  } else if (warp == 3) {
    // ------------------------------------------------------------ W producer (this CTA's half of N)
    if (lane == 0) {
      if (rank == 0) mbar_expect_tx(bar(WH_FULL), 2u * 16384u);
      for (int pl = 0; pl < 2; ++pl)
        for (int kb = 0; kb < 2; ++kb)
          tma_load_3d_pair(base + kWh + uint32_t(pl) * 8192u + uint32_t(kb) * 4096u, &tmWh, leader(WH_FULL), kb * BK,
                           int(rank) * 32, pl);
      uint32_t it = 0, lt = 0;
      for (int t = pair0; t < p.pairs; t += npairs, ++lt) {
        if (lt > 0) mbar_wait(bar(O_FULL), (lt - 1) & 1u);
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int o = int(it % kNO);
          mbar_wait(bar(OP_EMPTY + o), ((it / kNO) & 1u) ^ 1u);
          const uint32_t b_hi = base + kOpB + uint32_t(o) * kOperand;
          if (rank == 0) mbar_expect_tx(bar(OP_FULL + o), 2 * (kTerms > 1 ? 2 : 1) * kPlaneB);
          const int nrow = int(rank) * (kN / 2);
          tma_load_3d_pair(b_hi, &tmW, leader(OP_FULL + o), kb * BK, nrow, 0);
          if constexpr (kTerms > 1) tma_load_3d_pair(b_hi + kPlaneB, &tmW, leader(OP_FULL + o), kb * BK, nrow, 1);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader)
    // The whole warp runs the loop (warp-uniform state and descriptors); one
    // elected lane issues each batch of tcgen05.mma and its commit.
    if (rank == 0) {
      constexpr uint32_t m256 = uint32_t(BM >> 4) << 24;
      constexpr uint32_t idQKV = instr_desc_tf32(kN) + m256, idS = instr_desc_tf32(256) + m256,
                         idC = instr_desc_tf32(128) + m256, idZ = instr_desc_tf32(kDK) + m256;
      uint32_t it = 0, lt = 0;
      bool wh = false;
      for (int t = pair0; t < p.pairs; t += npairs, ++lt) {
        const uint32_t ph = lt & 1u;
        // The last pair's C accumulator [0,128) was drained before C_READY and its Z
        // accumulator lives at [448,512): the projection may overwrite [0,192) at once
        // (tcgen05.mma executes in issue order, after the last pair's Z MMA).
        if (lane == 0) TL(lt, 0);
        // phase 1: [Q|K|V] = X · W
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int o = int(it % kNO);
          mbar_wait(bar(OP_FULL + o), (it / kNO) & 1u);
          if (lane == 0 && kb == 0) TL(lt, 2);
          tc_fence_after();
          const uint32_t a_hi = tmem + kTStage + uint32_t(o) * 64u, a_lo = a_hi + 32u;
          const uint32_t b_hi = base + kOpB + uint32_t(o) * kOperand, b_lo = b_hi + kPlaneB;
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk)
              mma3<kTerms>(tmem, a_hi + uint32_t(kk) * 8u, a_lo + uint32_t(kk) * 8u, b_hi + uint32_t(kk) * 32u,
                           b_lo + uint32_t(kk) * 32u, idQKV, (kb | kk) ? 1u : 0u);
            mma_commit_pair(bar(OP_EMPTY + o));
          }
          __syncwarp();
        }
        if (lane == 0) TL(lt, 3);
        if (elect_one()) mma_commit_pair(bar(ACC_FULL));
        __syncwarp();
        // S = Q Kᵀ (K = 64)
        mbar_wait(bar(A_READY), ph);
        if (lane == 0) TL(lt, 4);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < kDK / 8; ++kk) {
            const uint32_t kbo = uint32_t(kk >> 2) * 16384u + uint32_t(kk & 3) * 32u;
            mma3<kTerms>(tmem, tmem + kTQ + uint32_t(kk) * 8u, tmem + kTQ + 64u + uint32_t(kk) * 8u,
                         base + kKop + kbo, base + kKop + 32768u + kbo, idS, kk ? 1u : 0u);
          }
          mma_commit_pair(bar(S_FULL));
        }
        __syncwarp();
        // C = P V (K = 128 keys)
        mbar_wait(bar(V_READY), ph);
        mbar_wait(bar(P_READY), ph);
        if (lane == 0) TL(lt, 5);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < kS / 8; ++kk) {
            const uint32_t kbo = uint32_t(kk >> 2) * 8192u + uint32_t(kk & 3) * 32u;
            mma3<kTerms>(tmem, tmem + kTQ + uint32_t(kk) * 8u, tmem + kTQ + 128u + uint32_t(kk) * 8u,
                         base + kVop + kbo, base + kVop + 32768u + kbo, idC, kk ? 1u : 0u);
          }
          mma_commit_pair(bar(O_FULL));
        }
        __syncwarp();
        // Z = C Wh (K = 64)
        if (!wh) {
          mbar_wait(bar(WH_FULL), 0);
          wh = true;
        }
        mbar_wait(bar(C_READY), ph);
        if (lane == 0) TL(lt, 6);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < kDK / 8; ++kk) {
            const uint32_t kbo = uint32_t(kk >> 2) * 4096u + uint32_t(kk & 3) * 32u;
            mma3<kTerms>(tmem + kTZ, tmem + kTQ + uint32_t(kk) * 8u, tmem + kTQ + 64u + uint32_t(kk) * 8u,
                         base + kWh + kbo, base + kWh + 8192u + kbo, idZ, kk ? 1u : 0u);
          }
          mma_commit_pair(bar(Z_FULL));
        }
        __syncwarp();
      }
    }
  } else if (warp >= 4 && warp < 12) {
    // ------------------------------------------------------------ converters (phase 1) / row warps (phase 2)
    const int q = warp & 3, g = (warp - 4) >> 2, row = q * 32 + lane;
    const uint32_t lane_base = tmem + (uint32_t(q * 32) << 16);
    const uint32_t mine = base + kExch + uint32_t(q * 2 + g) * 256u + uint32_t(lane) * 4u;
    const uint32_t other = base + kExch + uint32_t(q * 2 + (g ^ 1)) * 256u + uint32_t(lane) * 4u;
    const float sl = p.scale * 1.4426950408889634f;
    const int col0 = int(rank) * kS;  // this CTA's block of S (its own keys)
    // one K-block of X rows -> TMEM A stage (iteration `i` of the stage rings)
    auto convert = [&](uint32_t i, int kb) {
      (void)g;
      const int s = int(i % kNS), o = int(i % kNO);
      mbar_wait(bar(ST_FULL + s), (i / kNS) & 1u);
      mbar_wait(bar(OP_EMPTY + o), ((i / kNO) & 1u) ^ 1u);
      tc_fence_after();
      const uint32_t sa = base + kU + uint32_t(s) * kStaging;
      const uint32_t ta = lane_base + kTStage + uint32_t(o) * 64u;
      (void)kb;
#pragma unroll
      for (int hh = 0; hh < (HS_DBG_HEAD_NOCONV ? 0 : 2); ++hh) {
        uint32_t x[16], hi[16], lo[16];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float4 v = lds128(sa + sw128(row, 4 * hh + c));
          x[4 * c] = __float_as_uint(v.x); x[4 * c + 1] = __float_as_uint(v.y);
          x[4 * c + 2] = __float_as_uint(v.z); x[4 * c + 3] = __float_as_uint(v.w);
        }
        split_row16<kTerms>(x, hi, lo);
        tmem_st16(ta + uint32_t(16 * hh), hi);
        if constexpr (kTerms > 1) tmem_st16(ta + 32u + uint32_t(16 * hh), lo);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(bar(ST_EMPTY + s));
        mbar_arrive_cluster(leader(OP_FULL + o));
      }
    };
    uint32_t it = 0, lt = 0;
    // K-blocks of the current pair this group converted during the last pair's phase 2
    bool pre0 = false, pre3 = false;
    int pre0k = 0;  // which K-block went to stage 0 early
    for (int t = pair0; t < p.pairs; t += npairs, ++lt) {
      const uint32_t ph = lt & 1u;
      // ---- phase 1: split this CTA's X rows into the TMEM A stages (every other K-block)
      for (int kb = 0; kb < nk; ++kb, ++it) {
        if (int(it % kConv) != g || (kb == pre0k && pre0) || (kb == 3 && pre3)) continue;
        convert(it, kb);
      }
      pre0 = pre3 = false;
      // ---- phase 2 (A): operands of S = Q Kᵀ and C = P V, split across 12 warps:
      //      g = 0: Q (64 columns) -> tf32 hi [256, 320) / lo [320, 384) in TMEM
      //      g = 1: K -> K-major smem hi/lo, and Vᵀ for d in [0, 32)
      //      (warps 12-15: Vᵀ for d in [32, 64))
      if (warp == 4 && lane == 0) TL(lt, 7);
      mbar_wait(bar(ACC_FULL), ph);
      if (warp == 4 && lane == 0) TL(lt, 8);
      tc_fence_after();
      if (g == 0) {  // Q -> TMEM A operand
#pragma unroll 1
        for (int cb = 0; cb < 2; ++cb) {
          uint32_t r[32], hi[16], lo[16];
          tmem_ld32(lane_base + uint32_t(cb * 32), r);
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            split_row16<kTerms>(r + 16 * hh, hi, lo);
            const uint32_t col = kTQ + uint32_t(cb * 32 + hh * 16);
            tmem_st16(lane_base + col, hi);
            tmem_st16(lane_base + col + 64u, lo);
          }
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(leader(A_READY));
      } else {  // K, then half of Vᵀ
        store_k_operand(base, lane_base, row);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(leader(A_READY));
        store_vt_operand(base, lane_base, q, lane, 0);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(leader(V_READY));
      }
      // ---- (B) softmax over this CTA's S block, columns [col0 + 64g, +64) in registers
      mbar_wait(bar(S_FULL), ph);
      if (warp == 4 && lane == 0) TL(lt, 9);
      tc_fence_after();
      uint32_t r0[32], r1[32];
      tmem_ld32_nowait(lane_base + uint32_t(col0 + g * 64), r0);
      tmem_ld32_nowait(lane_base + uint32_t(col0 + g * 64 + 32), r1);
      tmem_ld_wait(r0);
      tmem_ld_dep(r1);
      const bool full = p.S >= kS;  // warp-uniform: no key masking
      float mx = full ? row_max<false>(r0, r1, 0, p.S, p.scale) : row_max<true>(r0, r1, g * 64, p.S, p.scale);
      sts32(mine, mx);
      named_bar(1u + uint32_t(q), 64u);
      mx = fmaxf(mx, lds32(other));
      const float ml = mx * 1.4426950408889634f;
      const float sum = full ? row_exp<false>(r0, r1, 0, p.S, sl, ml) : row_exp<true>(r0, r1, g * 64, p.S, sl, ml);
      sts32(mine + 128u, sum);
      named_bar(1u + uint32_t(q), 64u);
      const float s_other = lds32(other + 128u);
      const float inv = 1.f / (g == 0 ? sum + s_other : s_other + sum);
#pragma unroll
      for (int hh = 0; hh < 4; ++hh) {
        uint32_t hi[16], lo[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const float x = __uint_as_float(hh < 2 ? r0[(hh & 1) * 16 + e] : r1[(hh & 1) * 16 + e]) * inv;
          const float h = tf32_rna(x);
          hi[e] = __float_as_uint(h);
          lo[e] = __float_as_uint(x - h);
        }
        const uint32_t col = kTQ + uint32_t(g * 64 + hh * 16);
        tmem_st16(lane_base + col, hi);
        tmem_st16(lane_base + col + 128u, lo);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(leader(P_READY));
      // The next pair's first K-block goes to A stage 0 = TMEM [192, 256), part of S:
      // free once every warp of this lane quarter has read S (both passed the
      // exchange barriers above). Convert it while P·V runs (its X tile was loaded
      // after S_FULL into the K operand's smem).
      if constexpr (kConv == 2) {
        if (t + npairs < p.pairs && int(it & 1u) == g && it % kNO == 0) {
          convert(it, 0);
          pre0 = true;
          pre0k = 0;
        }
      } else {
        // the first of the next pair's K-blocks 0-2 that maps to stage 0 (group 0 owns
        // it, as kNO == kConv), if its X stage lies in the K operand's smem
        for (uint32_t j = 0; j < 3 && int(j) < nk; ++j)
          if ((it + j) % kNO == 0) {
            if (t + npairs < p.pairs && g == 0 && (it + j) % kNS < 4) {
              convert(it + j, int(j));
              pre0 = true;
              pre0k = int(j);
            }
            break;
          }
      }
      // ---- (C) C columns [64r + 32g, +32) -> tf32 hi [256, 320) / lo [320, 384)
      mbar_wait(bar(O_FULL), ph);
      if (warp == 4 && lane == 0) TL(lt, 10);
      tc_fence_after();
      {
        uint32_t r[32], hi[16], lo[16];
        tmem_ld32(lane_base + uint32_t(int(rank) * kDK + g * 32), r);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          split_row16<kTerms>(r + 16 * hh, hi, lo);
          const uint32_t col = kTQ + uint32_t(g * 32 + hh * 16);
          tmem_st16(lane_base + col, hi);
          tmem_st16(lane_base + col + 64u, lo);
        }
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(leader(C_READY));
      // The next pair's K-block 3 goes to A stage 3 = TMEM [384, 448), P lo's
      // columns: free once P·V has run (O_FULL, waited above). Its X tile was
      // loaded after S_FULL like the first ones.
      if constexpr (kConv == 2) {
        if (t + npairs < p.pairs && nk > 3 && int((it + 3u) & 1u) == g && it % kNO == 0) {
          convert(it + 3u, 3);
          pre3 = true;
        }
      }
      // The next pair's A stages 1-2 overlap C hi/lo [256, 384): convert only after
      // the Z MMA has read them. The Z accumulator is drained by warps 12-15.
      mbar_wait(bar(Z_FULL), ph);
      if (warp == 4 && lane == 0) TL(lt, 11);
    }
  } else if (warp >= 12) {
    // ------------------------------------------------------------ operand / Z warps (phase 2)
    // (HS_HEAD_CONV3: also converter group 2 in phase 1)
    const int q = warp & 3;
    const uint32_t lane_base = tmem + (uint32_t(q * 32) << 16);
    const uint32_t stage = base + kEpi + uint32_t(q) * 8192u;
    uint32_t lt = 0, it = 0;
    const int row = q * 32 + lane;
    (void)row;
    for (int t = pair0; t < p.pairs; t += npairs, ++lt) {
      const uint32_t ph = lt & 1u;
      const int inst = 2 * t + int(rank);
      if constexpr (kConv == 3) {
        for (int kb = 0; kb < nk; ++kb, ++it) {
          if (it % 3u != 2u) continue;
          const int s = int(it % kNS), o = int(it % kNO);
          mbar_wait(bar(ST_FULL + s), (it / kNS) & 1u);
          mbar_wait(bar(OP_EMPTY + o), ((it / kNO) & 1u) ^ 1u);
          tc_fence_after();
          const uint32_t sa = base + kU + uint32_t(s) * kStaging;
          const uint32_t ta = lane_base + kTStage + uint32_t(o) * 64u;
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            uint32_t x[16], hi[16], lo[16];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const float4 v = lds128(sa + sw128(row, 4 * hh + c));
              x[4 * c] = __float_as_uint(v.x); x[4 * c + 1] = __float_as_uint(v.y);
              x[4 * c + 2] = __float_as_uint(v.z); x[4 * c + 3] = __float_as_uint(v.w);
            }
            split_row16<kTerms>(x, hi, lo);
            tmem_st16(ta + uint32_t(16 * hh), hi);
            if constexpr (kTerms > 1) tmem_st16(ta + 32u + uint32_t(16 * hh), lo);
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(bar(ST_EMPTY + s));
            mbar_arrive_cluster(leader(OP_FULL + o));
          }
        }
      }
      mbar_wait(bar(ACC_FULL), ph);
      tc_fence_after();
      if (warp == 12 && lane == 0) TL(lt, 12);
      store_vt_operand(base, lane_base, q, lane, 1);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (warp == 12 && lane == 0) TL(lt, 13);
      if (lane == 0) mbar_arrive_cluster(leader(V_READY));
      // Z accumulator [448, 512) -> SW128 staging (2 x [32 rows][32 cols]) -> TMA store
      mbar_wait(bar(Z_FULL), ph);
      tc_fence_after();
#pragma unroll 1
      for (int cb = 0; cb < 2; ++cb) {
        uint32_t r[32];
        tmem_ld32(lane_base + kTZ + uint32_t(cb * 32), r);
        const uint32_t buf = stage + uint32_t(cb) * 4096u;
        if (lt > 0) {  // the last pair's store of this buffer has read it
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          __syncwarp();
        }
#pragma unroll
        for (int c = 0; c < 8; ++c)
          sts128(buf + uint32_t(lane) * 128u + (uint32_t(c ^ (lane & 7)) << 4),
                 make_float4(__uint_as_float(r[4 * c]), __uint_as_float(r[4 * c + 1]), __uint_as_float(r[4 * c + 2]),
                             __uint_as_float(r[4 * c + 3])));
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          if (inst < p.batch) tma_store_3d(&tmZ, buf, cb * 32, q * 32, inst);
          else asm volatile("cp.async.bulk.commit_group;" ::: "memory");  // keep the group count per buffer
        }
      }
      tc_fence_before();
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

}  // namespace

}  // namespace hs

// timing experiment only: copy the debug timeline (8 x 16 clock64 stamps) to host
extern "C" int hs_debug_head_timeline(long long* out) {
#if HS_DBG_TIMELINE
  return cudaMemcpyFromSymbol(out, hs::g_head_timeline, sizeof(long long) * 128) == cudaSuccess ? 0 : 1;
#else
  (void)out;
  return 1;
#endif
}

namespace hs {

bool head_fused_supported(const HeadArgs& a) {
  if (a.S < 1 || a.S > kS || a.dk != kDK || a.D < BK || a.D % BK || a.batch < 1 || !a.Wqkv || !a.Wh) return false;
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  if (!al16(a.X) || !al16(a.Z) || !al16(a.Wqkv) || !al16(a.Wh)) return false;
  const int64_t ld = a.ldz ? a.ldz : kDK;
  if ((a.sX | a.sZ | ld) & 3) return false;
  return encode_fn() != nullptr;
}

cudaError_t head_fused(const HeadArgs& a, int terms, cudaStream_t s) {
  if (!head_fused_supported(a)) return cudaErrorInvalidValue;
  auto kernel = terms > 1 ? head_pair_kernel<3> : head_pair_kernel<1>;
  static std::once_flag once3, once1;
  static cudaError_t err3 = cudaSuccess, err1 = cudaSuccess;
  std::call_once(terms > 1 ? once3 : once1, [&] {
    (terms > 1 ? err3 : err1) = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
  });
  if (cudaError_t e = terms > 1 ? err3 : err1) return e;
  const uint64_t S = uint64_t(a.S), D = uint64_t(a.D), B = uint64_t(a.batch);
  const uint64_t ldz = uint64_t(a.ldz ? a.ldz : kDK);
  CUtensorMap mX, mW, mWh, mZ;
  bool ok = make_map(&mX, a.X, D, S, B, D * 4, uint64_t(a.sX ? a.sX : S * D) * 4, BK, BM, true) &&
            make_map(&mW, a.Wqkv, D, kN, 2, D * 4, uint64_t(kN) * D * 4, BK, kN / 2, true) &&
            make_map(&mWh, a.Wh, kDK, kDK, 2, kDK * 4, uint64_t(kDK * kDK) * 4, BK, kDK / 2, true) &&
            make_map(&mZ, a.Z, kDK, S, B, ldz * 4, uint64_t(a.sZ ? a.sZ : S * ldz) * 4, 32, 32, true);
  if (!ok) return cudaErrorInvalidValue;
  HeadParams p{a.S, a.D, a.batch, (a.batch + 1) / 2, a.scale};
  const int max_pairs = num_sms() / 2;
  const int pairs = p.pairs < max_pairs ? p.pairs : max_pairs;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, mX, mW, mWh, mZ, p);
}

}  // namespace hs
