// Whole transformer head as one sm_100a launch (HS_OP_HEAD):
//
//   Q | K | V = X · [Wq | Wk | Wv]         X: [S, D]   W*: [D, 64]   (resident, pre-split)
//   Z         = softmax_row(s · Q Kᵀ) · V · Wh              Wh: [64, 64] (resident, pre-split)
//
// which is the head component of the encoder DAG (SURVEY.md §8 C3:
// three projection GEMMs, transpose, QKᵀ, softmax, P·V, C·W_h) after the engine's
// launch rewrites. Q, K, V, S, P and C never leave the SM. Every product is 3xTF32
// on tcgen05 (hi/lo splits, lo·hi + hi·lo + hi·hi).
//
// A cluster of two CTAs (one TPC) per pair of instances, persistent over pairs,
// and two pairs in flight: while the tensor cores run the Q/K/V projection of
// pair i+1, the attention of pair i runs beside it.
//   projection  cta_group::2, M = 256 (each CTA its own instance's 128 rows), N = 192,
//               K-blocks of 16 X columns: X tile -> tf32 hi/lo in a TMEM A stage (32
//               columns) by the converter warps; W planes K-major SWIZZLE_128B in
//               K-blocks of 32, each CTA holding half of N (96 rows): the pair halves
//               each SM's shared-memory traffic for W, which a single CTA at N = 192
//               cannot sustain
//   attention   cta_group::1 per CTA on its own instance (no cross-instance blocks):
//               S = Q Kᵀ (N = 128, Q hi/lo in TMEM, K hi/lo in smem), softmax in
//               registers, C = P V (N = 64, P hi/lo in TMEM, Vᵀ hi/lo in smem),
//               Z = C Wh (N = 64, C hi/lo in TMEM, Wh planes in smem)
// Two issuer warps per CTA feed one tensor pipe: the leader's warp 1 issues the
// projection, and warp 2 of each CTA issues that CTA's attention in pair order, so
// neither stream waits on the other's barriers (profiles/mix_probe.cu: cta_group::1
// and ::2 MMAs side by side in one cluster kernel, from one thread or from two
// warps, are exact).
//
// Warp roles (512 threads per CTA):
//   warp 0      TMA: this CTA's X tiles (+ L2 prefetch of its next instance's X)
//   warp 1      MMA issuer: the projection (leader only)
//   warp 2      TMEM allocator (512 columns, cta_group::2); then MMA issuer of this
//               CTA's attention (S, P·V, Z) and TMA of the Wh planes
//   warp 3      TMA: this CTA's half of the Wq|Wk|Wv planes
//   warps 4-7   converters: X tile -> tf32 hi/lo -> TMEM A stage (lane quarter = warp % 4)
//   warps 8-15  attention (quarter q = warp % 4, half g = (warp - 8) / 4): extraction
//               (Q -> TMEM hi/lo, K / Vᵀ -> smem hi/lo), softmax, P -> TMEM, C -> TMEM
//               hi/lo, Z -> global
//
// TMEM columns (each CTA): [0,192) projection accumulator Q|K|V · [192,256) 2 A
// stages · [256,384) Q hi|lo -> P hi|lo of keys 0-63 -> P hi|lo of keys 64-127 -> C
// hi|lo · [384,512) S -> C accumulator [384,448) + Z accumulator [448,512).
//
// Measured (profiles/head_probe.py): 80 us per 512-instance launch (round 1: 100 us;
// one issuer warp for both streams: 88 us). Per pair (profiles/head_timeline.py,
// ~32k cycles): the tensor pipe holds 18.4k cycles of projection and ~3.8k of
// attention MMAs (the narrow shapes run at full rate, profiles/mma_rate.cu); the rest
// is the two-stage A ring's converter round trip (~11k cycles of issuer waits) and the
// accumulator hand-over between pairs (~5k), both bounded by TMEM (512 columns) and
// shared memory (224 KB) rather than by the X / W rings (deeper rings: no change).
#include <mutex>

#include "kernels.cuh"
#include "launch.cuh"
#include "tc_common.cuh"

#ifndef HS_DBG_TIMELINE
#define HS_DBG_TIMELINE 0
#endif
// timing experiments only (wrong results): skip the X split (converters only signal),
// or the attention (no QKᵀ / P·V / softmax / Z; the accumulator is released at once)
#ifndef HS_DBG_HEAD_NOCONV
#define HS_DBG_HEAD_NOCONV 0
#endif
#ifndef HS_DBG_HEAD_NOPROJ  // timing experiment only: no projection MMAs (commits only)
#define HS_DBG_HEAD_NOPROJ 0
#endif
#ifndef HS_HEAD_PREFETCH_AHEAD  // pairs of X prefetched into L2 ahead of the current one
#define HS_HEAD_PREFETCH_AHEAD 1
#endif
#ifndef HS_DBG_HEAD_XSRC
#define HS_DBG_HEAD_XSRC 0
#endif
#ifndef HS_DBG_HEAD_NOATT
#define HS_DBG_HEAD_NOATT 0
#endif

namespace hs {

#if HS_DBG_TIMELINE
// timing experiment only (profiles/head_timeline.py): CTA 0, first 8 pair iterations
// x 32 slots: clock stamps (low 32 bits), and cycles spent in selected waits (summed).
// Accumulated in shared memory (a global read-modify-write would add its own latency
// to every measured interval) and copied out at the end.
__device__ long long g_head_timeline[8 * 32];
#define TL(t, k)                                                           \
  do {                                                                     \
    if (blockIdx.x == 0 && (t) < 8) s_tl[(t) * 32 + (k)] = uint32_t(clock64()); \
  } while (0)
#define TW(t, k, expr)                                                          \
  do {                                                                          \
    const long long _c0 = clock64();                                            \
    expr;                                                                       \
    const long long _c1 = clock64();                                            \
    if (blockIdx.x == 0 && (t) < 8 && lane == 0) s_tl[(t) * 32 + (k)] += uint32_t(_c1 - _c0); \
  } while (0)
#define TADD(t, k, v)                                              \
  do {                                                             \
    if (blockIdx.x == 0 && (t) < 8 && lane == 0) s_tl[(t) * 32 + (k)] += uint32_t(v); \
  } while (0)
#else
#define TL(t, k) \
  do {           \
  } while (0)
#define TW(t, k, expr) expr
#define TADD(t, k, v) \
  do {                \
  } while (0)
#endif

namespace {

using namespace tc;

constexpr int kS = 128, kDK = 64, kN = 3 * kDK;  // rows, head width, projection width
constexpr int kThreads = 512;
// HS_HEAD_RZ: tcgen05 kind::tf32 reads an fp32 operand by truncating its low 13
// mantissa bits (profiles/tf32_trunc_probe.cu: round-toward-zero, from shared memory
// and from TMEM alike), so a raw fp32 X tile is already the hi term of an exact
// split x = rz(x) + (x - rz(x)). The projection's hi·W products read the TMA-landed X
// tile straight from shared memory; only lo = rna(x - rz(x)) goes through the
// converters into a TMEM A stage (16 columns instead of 32: half the TMEM stores, and
// four stages where the hi|lo split fit two). The X slot then stays live until the
// MMAs that read it complete (their commit frees it).
#ifndef HS_HEAD_RZ
#define HS_HEAD_RZ 0
#endif
#ifndef HS_HEAD_WK
#define HS_HEAD_WK 32
#endif
#ifndef HS_HEAD_NW
#define HS_HEAD_NW (HS_HEAD_RZ ? 2 : 3)
#endif
#ifndef HS_HEAD_XK
#define HS_HEAD_XK (HS_HEAD_RZ ? 32 : 16)
#endif
constexpr int kXK = HS_HEAD_XK;                  // X tile / A stage: 16 columns (SWIZZLE_64B) or 32 (SWIZZLE_128B)
static_assert(kXK == 16 || (kXK == 32 && HS_HEAD_RZ), "X tile width (32 only with lo-only A stages)");
constexpr int kWK = HS_HEAD_WK;                  // W stage: 32 columns (SWIZZLE_128B) = 2 A stages, or 16 (SWIZZLE_64B)
static_assert(kWK == 16 || kWK == 32, "W stage width");
#ifndef HS_HEAD_NA
#define HS_HEAD_NA 2
#endif
#ifndef HS_HEAD_NX
#define HS_HEAD_NX 3
#endif
constexpr int kNX = HS_HEAD_NX, kNW = HS_HEAD_NW, kNA = HS_HEAD_NA;  // ring depths
constexpr uint32_t kXTile = kS * kXK * 4;        // 8 KB
constexpr uint32_t kWPlane = (kN / 2) * kWK * 4;  // this CTA's 96 rows (12 KB at kWK = 32)
constexpr uint32_t kWStage = 2 * kWPlane;        // hi + lo
// shared memory (bytes from the 1024-aligned base)
constexpr uint32_t kXs = 0;
constexpr uint32_t kWs = kXs + kNX * kXTile;     // 24 KB
constexpr uint32_t kKop = kWs + kNW * kWStage;   // 96 KB: K hi/lo, 2 planes x 2 k-blocks x [128 keys][128 B]
constexpr uint32_t kVop = kKop + 65536;          // 160 KB: Vᵀ hi/lo, 2 planes x 4 k-blocks x [64 d][128 B]
constexpr uint32_t kBar = HS_DBG_HEAD_NOATT ? kKop : kVop + 65536;  // 224 KB
constexpr uint32_t kXch = kKop;                  // softmax row max / sum exchange (K consumed by then)
constexpr uint32_t kWh = kKop + 4096;            // Whᵀ hi/lo, 2 planes x 2 k-blocks x [64][128 B] (after S)
constexpr int kSmem = int(kBar) + 512 + 1024;
static_assert(kSmem <= 227 * 1024, "shared memory budget exceeded");

// TMEM columns
constexpr uint32_t kTQ = 0, kTK = 64, kTV = 128;  // projection accumulator
constexpr uint32_t kTA = 192;                     // A stages: lo 16 (HS_HEAD_RZ) or hi 16 | lo 16
constexpr uint32_t kAW = HS_HEAD_RZ ? kXK : 2 * kXK;  // columns per A stage
constexpr uint32_t kTOp = kTA + kAW * kNA;       // 128 columns: Q hi|lo -> P hi|lo (one key half) -> C hi|lo
constexpr uint32_t kTR = kTOp + 128;              // 128 columns: S -> C acc [kTR, +64) -> Z acc [kTR + 64, +64)
static_assert(HS_DBG_HEAD_NOATT || kTR + 128 <= 512, "TMEM columns");

enum Bar : uint32_t {
  XF = 0,               // [kNX] X tile landed (TMA tx)
  XE = XF + kNX,        // [kNX] X tile converted (4 local converter warps)
  WF = XE + kNX,        // [kNW] leader: both CTAs' W halves landed (TMA tx)
  WE = WF + kNW,        // [kNW] W stage consumed (leader's commit, multicast)
  AF = WE + kNW,        // [kNA] leader: both CTAs' A stages written (2 x 4 converter warps)
  AE = AF + kNA,        // [kNA] A stage consumed (leader's commit, multicast)
  ACC_FULL = AE + kNA,  // projection done (leader's commit, multicast)
  EXT_PAIR,             // leader: both CTAs extracted (2 x 8 attention warps)
  EXT,                  // this CTA extracted (8 warps): Q hi/lo in TMEM, K / Vᵀ in smem
  S_FULL,               // S = Q Kᵀ done (Q and K consumed)
  S_READ,               // ... read into registers (8 warps)
  WH_FULL,              // Wh planes landed (TMA tx)
  P0_READY,             // P hi|lo of keys 0-63 in TMEM (4 warps)
  PV0_DONE,             // C = P V over keys 0-63 done
  P1_READY,             // P hi|lo of keys 64-127 in TMEM (4 warps)
  C_FULL,               // C = P V done
  C_READY,              // C hi/lo in TMEM (8 warps)
  Z_FULL,               // Z = C Wh done
  TMEM_SLOT,
  kNumBars
};
static_assert(kNumBars * 8 <= 512, "barrier area");

struct HeadParams {
  int S, D, batch, pairs;
  float scale;
  float* Z;
  int64_t sZ, ldz;  // elements
};

// D (+)= A·B with A = a_hi + a_lo in TMEM, B = b_hi + b_lo in smem: lo·hi, hi·lo, hi·hi
template <int kTerms, bool kPair>
__device__ __forceinline__ void mma3(uint32_t d, uint32_t a_hi, uint32_t a_lo, uint64_t b_hi, uint64_t b_lo,
                                     uint32_t idesc, uint32_t first) {
  auto mma = [&](uint32_t a, uint64_t b, uint32_t acc) {
    if constexpr (kPair) mma_pair_tf32_ts(d, a, b, idesc, acc);
    else mma_tf32_ts(d, a, b, idesc, acc);
  };
  if constexpr (kTerms > 1) {
    mma(a_lo, b_hi, first);
    mma(a_hi, b_lo, 1u);
    mma(a_hi, b_hi, 1u);
  } else {
    mma(a_hi, b_hi, first);
  }
}

template <int kTerms>
__device__ __forceinline__ void split16(const uint32_t* r, uint32_t (&hi)[16], uint32_t (&lo)[16]) {
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const float x = __uint_as_float(r[e]);
    const float h = tf32_rna(x);
    hi[e] = __float_as_uint(h);
    lo[e] = __float_as_uint(tf32_lo(x, h));
  }
}

// 16 values -> hi / lo TMEM columns (hi at taddr, lo at taddr + lo_off)
template <int kTerms>
__device__ __forceinline__ void st_split16(uint32_t taddr, uint32_t lo_off, const uint32_t* r) {
  uint32_t hi[16], lo[16];
  split16<kTerms>(r, hi, lo);
  tmem_st16(taddr, hi);
  if constexpr (kTerms > 1) tmem_st16(taddr + lo_off, lo);
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

template <int kTerms>
__global__ void __launch_bounds__(kThreads, 1)
    head_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                const __grid_constant__ CUtensorMap tmWh, const __grid_constant__ CUtensorMap tmXp, HeadParams p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  auto bar = [&](uint32_t b) { return base + kBar + 8u * b; };
#if HS_DBG_TIMELINE
  __shared__ uint32_t s_tl[8 * 32];
  for (int i = threadIdx.x; i < 8 * 32; i += blockDim.x) s_tl[i] = 0;
#endif
  const uint32_t* tmem_slot_ptr =
      reinterpret_cast<const uint32_t*>(smem_raw + (bar(TMEM_SLOT) - smem_u32(smem_raw)));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int pair0 = int(cluster_id_x()), npairs = int(nclusters_x());
  const int nx = p.D / kXK, nw = p.D / kWK;
  auto leader = [&](uint32_t b) { return mapa_rank(bar(b), 0); };

  if (threadIdx.x == 0) {
    for (int s = 0; s < kNX; ++s) {
      mbar_init(bar(XF + s), 1);
      mbar_init(bar(XE + s), HS_HEAD_RZ ? 1 : 4);  // RZ: the leader's commit of the MMAs reading it
    }
    for (int s = 0; s < kNW; ++s) {
      mbar_init(bar(WF + s), 1);
      mbar_init(bar(WE + s), 1);
    }
    for (int a = 0; a < kNA; ++a) {
      mbar_init(bar(AF + a), 2 * 4);
      mbar_init(bar(AE + a), 1);
    }
    for (uint32_t b : {ACC_FULL, S_FULL, WH_FULL, PV0_DONE, C_FULL, Z_FULL}) mbar_init(bar(b), 1);
    mbar_init(bar(EXT_PAIR), 2 * 8);
    for (uint32_t b : {EXT, S_READ, C_READY}) mbar_init(bar(b), 8);
    for (uint32_t b : {P0_READY, P1_READY}) mbar_init(bar(b), 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (const CUtensorMap* m : {&tmX, &tmW, &tmWh, &tmXp})
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(bar(TMEM_SLOT)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  pdl_launch_dependents();  // PDL (launch.cuh)
  pdl_wait();
  const uint32_t tmem = *tmem_slot_ptr;

  if (warp == 0) {
    // ------------------------------------------------------------ X producer (this CTA's instance)
    if (lane == 0) {
      // Warm L2 with whole instances ahead of their X tiles: the tile ring keeps only
      // kNX x 8 KB in flight, too little to cover DRAM latency, while a prefetch of all
      // 16 128-byte row segments per row has no such limit (and the 64-byte tiles then
      // hit L2 instead of each fetching half of a DRAM line). X from L2 instead of DRAM
      // is worth ~10 % of the launch (profiles/README.md, HS_DBG_HEAD_XSRC).
      auto prefetch = [&](int t) {
        const int inst = 2 * t + int(rank);
        if (t < p.pairs && inst < p.batch)
          for (int kb = 0; kb < p.D / 32; ++kb) tma_prefetch_3d(&tmXp, kb * 32, 0, inst);
      };
      for (int a = 0; a < HS_HEAD_PREFETCH_AHEAD; ++a) prefetch(pair0 + a * npairs);
      uint32_t it = 0, lt = 0;
      for (int t = pair0; t < p.pairs; t += npairs, ++lt) {
        const int inst = 2 * t + int(rank);  // >= batch: zero-filled box
        prefetch(t + HS_HEAD_PREFETCH_AHEAD * npairs);
        for (int kb = 0; kb < nx; ++kb, ++it) {
          const int s = int(it % kNX);
          TW(lt, 12, mbar_wait(bar(XE + s), ((it / kNX) & 1u) ^ 1u));
#if HS_DBG_HEAD_XSRC == 2  // timing experiment only: no X loads
          mbar_arrive(bar(XF + s));
#else  // timing experiments only: HS_DBG_HEAD_XSRC == 1: every pair reads instance 0's X (L2-resident);
       // 3: every pair of a CTA re-reads its first instance
          mbar_expect_tx(bar(XF + s), kXTile);
          tma_load_3d(base + kXs + uint32_t(s) * kXTile, &tmX, bar(XF + s), kb * kXK, 0,
                      HS_DBG_HEAD_XSRC == 1 ? 0 : HS_DBG_HEAD_XSRC == 3 ? 2 * pair0 + int(rank) : inst);
#endif
        }
      }
    }
  } else if (warp == 3) {
    // ------------------------------------------------------------ W producer (this CTA's half of N)
    if (lane == 0) {
      uint32_t it = 0, lt = 0;
      for (int t = pair0; t < p.pairs; t += npairs, ++lt) {
        for (int kb = 0; kb < nw; ++kb, ++it) {
          const int s = int(it % kNW);
          TW(lt, 13, mbar_wait(bar(WE + s), ((it / kNW) & 1u) ^ 1u));
          if (rank == 0) mbar_expect_tx(bar(WF + s), 2u * (kTerms > 1 ? 2u : 1u) * kWPlane);
          const uint32_t dst = base + kWs + uint32_t(s) * kWStage;
          const int nrow = int(rank) * (kN / 2);
          tma_load_3d_pair(dst, &tmW, leader(WF + s), kb * kWK, nrow, 0);
          if constexpr (kTerms > 1) tma_load_3d_pair(dst + kWPlane, &tmW, leader(WF + s), kb * kWK, nrow, 1);
        }
      }
    }
  } else if (warp == 1 || warp == 2) {
    // ------------------------------------------------------------ MMA issuers
    // warp 1 (leader only): the projection; warp 2 (both CTAs): this CTA's attention
    // and the Wh planes. Each loop runs on the whole warp (warp-uniform state) and one
    // elected lane issues; every commit tracks the MMAs of its own issuing thread, and
    // the two streams share the tensor pipe (profiles/mix_probe.cu -DMIX_SPLIT=1).
    constexpr uint32_t idP = instr_desc_tf32(kN, 256), idS = instr_desc_tf32(kS), idC = instr_desc_tf32(kDK);
    auto kdesc = [&](int kk, int plane) {  // K operand: k-block kk/4 of d, 8-column step kk%4
      return smem_desc(base + kKop + uint32_t(plane) * 32768u + uint32_t(kk >> 2) * 16384u + uint32_t(kk & 3) * 32u);
    };
    auto vdesc = [&](int kk, int plane) {  // Vᵀ operand: k-block kk/4 of keys
      return smem_desc(base + kVop + uint32_t(plane) * 32768u + uint32_t(kk >> 2) * 8192u + uint32_t(kk & 3) * 32u);
    };
    auto whdesc = [&](int kk, int plane) {  // Whᵀ operand: k-block kk/4 of d
      return smem_desc(base + kWh + uint32_t(plane) * 16384u + uint32_t(kk >> 2) * 8192u + uint32_t(kk & 3) * 32u);
    };
    auto wdesc = [](uint32_t a) { return kWK == 32 ? smem_desc(a) : smem_desc_sw64(a); };
    uint32_t lt = 0;
    if (warp == 2) {
      // ---------------------------------------------------------- attention, in pair order
      for (int t = pair0; t < p.pairs && !HS_DBG_HEAD_NOATT; t += npairs, ++lt) {
        const uint32_t ph = lt & 1u;
        // S = Q hi|lo [kTOp, +128) x K -> kTR (N = 128), once this CTA has extracted
        TW(lt, 16, mbar_wait(bar(EXT), ph));
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < kDK / 8; ++kk)
            mma3<kTerms, false>(tmem + kTR, tmem + kTOp + uint32_t(kk) * 8u, tmem + kTOp + 64u + uint32_t(kk) * 8u,
                                kdesc(kk, 0), kdesc(kk, 1), idS, kk ? 1u : 0u);
          mma_commit(bar(S_FULL));
        }
        __syncwarp();
        // K consumed: the Wh planes land over the K operand
        TW(lt, 17, mbar_wait(bar(S_FULL), ph));
        if (lane == 0) {
          mbar_expect_tx(bar(WH_FULL), (kTerms > 1 ? 2u : 1u) * 16384u);
          for (int pl = 0; pl < (kTerms > 1 ? 2 : 1); ++pl)
            for (int kb = 0; kb < 2; ++kb)
              tma_load_3d(base + kWh + uint32_t(pl) * 16384u + uint32_t(kb) * 8192u, &tmWh, bar(WH_FULL), kb * 32, 0,
                          pl);
        }
        // C (+)= P·V per key half: P hi|lo [kTOp, +128) x Vᵀ k-blocks of those keys -> kTR
        for (int half = 0; half < 2; ++half) {
          if (half == 0) {
            TW(lt, 18, mbar_wait(bar(S_READ), ph));
            TW(lt, 18, mbar_wait(bar(P0_READY), ph));
          } else {
            TW(lt, 19, mbar_wait(bar(P1_READY), ph));
          }
          tc_fence_after();
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
              mma3<kTerms, false>(tmem + kTR, tmem + kTOp + uint32_t(kk) * 8u, tmem + kTOp + 64u + uint32_t(kk) * 8u,
                                  vdesc(8 * half + kk, 0), vdesc(8 * half + kk, 1), idC, (half | kk) ? 1u : 0u);
            mma_commit(bar(half ? C_FULL : PV0_DONE));
          }
          __syncwarp();
        }
        // Z = C hi|lo x Wh -> kTR + 64
        TW(lt, 20, mbar_wait(bar(WH_FULL), ph));
        TW(lt, 20, mbar_wait(bar(C_READY), ph));
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < kDK / 8; ++kk)
            mma3<kTerms, false>(tmem + kTR + 64u, tmem + kTOp + uint32_t(kk) * 8u,
                                tmem + kTOp + 64u + uint32_t(kk) * 8u, whdesc(kk, 0), whdesc(kk, 1), idC,
                                kk ? 1u : 0u);
          mma_commit(bar(Z_FULL));
        }
        __syncwarp();
      }
    } else if (rank == 0) {
      // ---------------------------------------------------------- projection (leader)
      uint32_t ia = 0, iw = 0;
      for (int t = pair0; t < p.pairs; t += npairs, ++lt) {
        // both CTAs have read the accumulator out: the next projection may overwrite it
        if (lt > 0) TW(lt, 6, mbar_wait(bar(EXT_PAIR), (lt - 1) & 1u));
        if (lane == 0) TL(lt, 0);
        for (int kb = 0; kb < nw; ++kb, ++iw) {
          const int w = int(iw % kNW);
          TW(lt, 8, mbar_wait(bar(WF + w), (iw / kNW) & 1u));
#pragma unroll 1
          for (int h = 0; h < kWK / kXK; ++h, ++ia) {
            const int a = int(ia % kNA);
            TW(lt, 9, mbar_wait(bar(AF + a), (ia / kNA) & 1u));
            tc_fence_after();
#if HS_DBG_TIMELINE
            const long long c_iss0 = clock64();
#endif
            if (elect_one()) {
              const uint32_t b = base + kWs + uint32_t(w) * kWStage + uint32_t(h) * uint32_t(kXK * 4);
              const uint32_t ta = tmem + kTA + uint32_t(a) * kAW;
#if HS_HEAD_RZ
              // lo·W_hi from the TMEM A stage; hi·W_lo and hi·W_hi read the raw X tile
              // (each CTA's own 128 rows, same slot offset in both CTAs)
              const int x = int(ia % kNX);
              const uint32_t xa = base + kXs + uint32_t(x) * kXTile;
#pragma unroll
              for (int kk = 0; kk < kXK / 8 && !HS_DBG_HEAD_NOPROJ; ++kk) {
                const uint32_t first = (kb | h | kk) ? 1u : 0u;
                const uint64_t xd = kXK == 32 ? smem_desc(xa + uint32_t(kk) * 32u) : smem_desc_sw64(xa + uint32_t(kk) * 32u);
                if constexpr (kTerms > 1) {
                  mma_pair_tf32_ts(tmem + kTQ, ta + uint32_t(kk) * 8u, wdesc(b + uint32_t(kk) * 32u), idP, first);
                  mma_pair_tf32_ss(tmem + kTQ, xd, wdesc(b + kWPlane + uint32_t(kk) * 32u), idP, 1u);
                  mma_pair_tf32_ss(tmem + kTQ, xd, wdesc(b + uint32_t(kk) * 32u), idP, 1u);
                } else {
                  mma_pair_tf32_ss(tmem + kTQ, xd, wdesc(b + uint32_t(kk) * 32u), idP, first);
                }
              }
              mma_commit_pair(bar(XE + x));
#else
#pragma unroll
              for (int kk = 0; kk < kXK / 8 && !HS_DBG_HEAD_NOPROJ; ++kk)
                mma3<kTerms, true>(tmem + kTQ, ta + uint32_t(kk) * 8u, ta + 16u + uint32_t(kk) * 8u,
                                   wdesc(b + uint32_t(kk) * 32u), wdesc(b + kWPlane + uint32_t(kk) * 32u), idP,
                                   (kb | h | kk) ? 1u : 0u);
#endif
              mma_commit_pair(bar(AE + a));
              if (h == kWK / kXK - 1) mma_commit_pair(bar(WE + w));
            }
            __syncwarp();
#if HS_DBG_TIMELINE
            TADD(lt, 7, clock64() - c_iss0);
#endif
          }
        }
        if (elect_one()) mma_commit_pair(bar(ACC_FULL));
        __syncwarp();
        if (lane == 0) TL(lt, 1);
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ------------------------------------------------------------ converters: X tile -> TMEM A stage
    const int q = warp & 3, row = q * 32 + lane;
    const uint32_t lane_base = tmem + (uint32_t(q * 32) << 16);
    const uint32_t swz = kXK == 32 ? uint32_t(row & 7) : uint32_t((row >> 1) & 3);
    // The X tile is read and split into registers (and its staging slot released)
    // before waiting for the A stage to free up: only the TMEM stores and the signal
    // remain between the MMA's release of the stage and its next use.
    uint32_t it = 0, lt = 0;
    for (int t = pair0; t < p.pairs; t += npairs, ++lt) {
      for (int kb = 0; kb < nx; ++kb, ++it) {
        const int x = int(it % kNX), a = int(it % kNA);
#if HS_DBG_TIMELINE
        const long long c_x0 = clock64();
#endif
        mbar_wait(bar(XF + x), (it / kNX) & 1u);
#if HS_DBG_TIMELINE
        if (q == 0) TADD(lt, 10, clock64() - c_x0);
#endif
        uint32_t hi[16], lo[kXK], dep = 0;
        if (!HS_DBG_HEAD_NOCONV) {
          const uint32_t src = base + kXs + uint32_t(x) * kXTile + uint32_t(row) * uint32_t(kXK * 4);
          uint32_t v[kXK];
#pragma unroll
          for (int c = 0; c < kXK / 4; ++c) {
            // SWIZZLE_64B: 16-byte chunk c of row r sits at chunk c ^ ((r >> 1) & 3);
            // SWIZZLE_128B: at chunk c ^ (r & 7)
            const float4 f = lds128(src + ((uint32_t(c) ^ swz) << 4));
            v[4 * c] = __float_as_uint(f.x);
            v[4 * c + 1] = __float_as_uint(f.y);
            v[4 * c + 2] = __float_as_uint(f.z);
            v[4 * c + 3] = __float_as_uint(f.w);
            dep ^= v[4 * c];  // one register of each LDS.128
          }
#if HS_HEAD_RZ
#pragma unroll
          for (int e = 0; e < kXK; ++e) {  // lo of the split the tensor core completes (hi = rz(x))
            const float xv = __uint_as_float(v[e]);
            lo[e] = __float_as_uint(tf32_rna(xv - __uint_as_float(v[e] & 0xFFFFE000u)));
          }
          (void)hi;
#else
          split16<kTerms>(v, hi, lo);
#endif
        }
#if !HS_HEAD_RZ
        // the staging slot goes back to TMA once this warp's loads have returned
        if (lane == 0) mbar_arrive_after(bar(XE + x), dep);
#else
        (void)dep;
#endif
#if HS_DBG_TIMELINE
        const long long c_a0 = clock64();
#endif
        mbar_wait(bar(AE + a), ((it / kNA) & 1u) ^ 1u);
#if HS_DBG_TIMELINE
        if (q == 0) TADD(lt, 11, clock64() - c_a0);
#endif
        tc_fence_after();
#if HS_DBG_TIMELINE
        const long long c_conv0 = clock64();
#endif
        if (!HS_DBG_HEAD_NOCONV) {
          const uint32_t ta = lane_base + kTA + uint32_t(a) * kAW;
#if HS_HEAD_RZ
          if constexpr (kTerms > 1) {
            tmem_st16(ta, *reinterpret_cast<const uint32_t(*)[16]>(lo));
            if constexpr (kXK == 32) tmem_st16(ta + 16u, *reinterpret_cast<const uint32_t(*)[16]>(lo + 16));
          }
#else
          tmem_st16(ta, hi);
          if constexpr (kTerms > 1) tmem_st16(ta + 16u, lo);
#endif
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
#if HS_DBG_TIMELINE
        const long long c_conv1 = clock64();
#endif
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          // relaxed: the stage's TMEM stores are complete (tcgen05.wait::st above); a
          // release arrive at cluster scope costs ~1k cycles per stage in this thread
          asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(leader(AF + a))
                       : "memory");
        }
#if HS_DBG_TIMELINE
        const long long c_conv2 = clock64();
        if (q == 0) {
          TADD(lt, 14, c_conv1 - c_conv0);
          TADD(lt, 15, c_conv2 - c_conv1);
        }
#endif
      }
    }
  } else if (warp >= 8) {
    // ------------------------------------------------------------ attention warps (this CTA's instance)
    const int q = warp & 3, g = (warp - 8) >> 2, row = q * 32 + lane;
    const uint32_t lane_base = tmem + (uint32_t(q * 32) << 16);
    const uint32_t mine = base + kXch + uint32_t(q * 2 + g) * 256u + uint32_t(lane) * 4u;
    const uint32_t other = base + kXch + uint32_t(q * 2 + (g ^ 1)) * 256u + uint32_t(lane) * 4u;
    const float sl = p.scale * 1.4426950408889634f;
    const bool full = p.S >= kS;  // uniform: no key masking
    uint32_t lt = 0;
    for (int t = pair0; t < p.pairs; t += npairs, ++lt) {
      const uint32_t ph = lt & 1u;
      const int inst = 2 * t + int(rank);
      // ---- extraction (the accumulator is free for the next projection afterwards)
      mbar_wait(bar(ACC_FULL), ph);
      tc_fence_after();
      if (warp == 8 && lane == 0) TL(lt, 2);
      if (!HS_DBG_HEAD_NOATT) {
        uint32_t r[32];
        // Q columns [32g, 32g+32) -> tf32 hi [256 + 32g) / lo [320 + 32g)
        tmem_ld32(lane_base + kTQ + uint32_t(32 * g), r);
        st_split16<kTerms>(lane_base + kTOp + uint32_t(32 * g), 64u, r);
        st_split16<kTerms>(lane_base + kTOp + uint32_t(32 * g + 16), 64u, r + 16);
        if (warp == 8 && lane == 0) TL(lt, 24);
        // K row (key = row), d in [32g, 32g+32) -> K-major SW128 k-block g (hi, lo at +32 KB)
        tmem_ld32(lane_base + kTK + uint32_t(32 * g), r);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const float4 x = make_float4(__uint_as_float(r[4 * c]), __uint_as_float(r[4 * c + 1]),
                                       __uint_as_float(r[4 * c + 2]), __uint_as_float(r[4 * c + 3]));
          const float4 h = make_float4(tf32_rna(x.x), tf32_rna(x.y), tf32_rna(x.z), tf32_rna(x.w));
          const uint32_t dst = base + kKop + uint32_t(g) * 16384u + sw128(row, c);
          sts128(dst, h);
          if constexpr (kTerms > 1) sts128(dst + 32768u, tf32_lo4(x, h));
        }
        if (warp == 8 && lane == 0) TL(lt, 25);
        // V row (key = row: k-block q, key lane), d in [32g, 32g+32) -> Vᵀ K-major SW128 [64 d][32 keys]
        tmem_ld32(lane_base + kTV + uint32_t(32 * g), r);
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float x = __uint_as_float(r[j]);
          const float h = tf32_rna(x);
          const uint32_t dst = base + kVop + uint32_t(q) * 8192u + sw128(32 * g + j, lane >> 2) + uint32_t(lane & 3) * 4u;
          sts32(dst, h);
          if constexpr (kTerms > 1) sts32(dst + 32768u, tf32_lo(x, h));
        }
        if (warp == 8 && lane == 0) TL(lt, 26);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(bar(EXT));
        mbar_arrive_cluster(leader(EXT_PAIR));
      }
      if (lane == 0 && (warp == 8 || warp == 15)) TL(lt, warp == 8 ? 27 : 28);
      if (HS_DBG_HEAD_NOATT) continue;
      // ---- softmax over keys [64g, 64g+64) of this row: S of this key half in registers
      mbar_wait(bar(S_FULL), ph);
      tc_fence_after();
      if (warp == 8 && lane == 0) TL(lt, 3);
      uint32_t r0[32], r1[32];
      tmem_ld32_nowait(lane_base + kTR + uint32_t(64 * g), r0);
      tmem_ld32_nowait(lane_base + kTR + uint32_t(64 * g + 32), r1);
      tmem_ld_wait(r0);
      tmem_ld_dep(r1);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar(S_READ));
      float mx = full ? row_max<false>(r0, r1, 0, p.S, p.scale) : row_max<true>(r0, r1, 64 * g, p.S, p.scale);
      sts32(mine, mx);
      named_bar(1u + uint32_t(q), 64u);
      mx = fmaxf(mx, lds32(other));
      const float ml = mx * 1.4426950408889634f;
      const float sum = full ? row_exp<false>(r0, r1, 0, p.S, sl, ml) : row_exp<true>(r0, r1, 64 * g, p.S, sl, ml);
      sts32(mine + 128u, sum);
      named_bar(1u + uint32_t(q), 64u);
      const float s_other = lds32(other + 128u);
      const float inv = 1.f / (g == 0 ? sum + s_other : s_other + sum);
      // P = e · inv of this key half -> hi [kTOp, +64) | lo [kTOp + 64, +64), once Q (key
      // half 0) or key half 0's P (key half 1) has been consumed
      if (g) mbar_wait(bar(PV0_DONE), ph);
      tc_fence_after();
      auto p_chunk = [&](const uint32_t(&r)[32], int off, int hh) {
        uint32_t v[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) v[e] = __float_as_uint(__uint_as_float(r[off + e]) * inv);
        st_split16<kTerms>(lane_base + kTOp + uint32_t(16 * hh), 64u, v);
      };
      p_chunk(r0, 0, 0);
      p_chunk(r0, 16, 1);
      p_chunk(r1, 0, 2);
      p_chunk(r1, 16, 3);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar(g ? P1_READY : P0_READY));
      // ---- C columns [32g, 32g+32) -> tf32 hi [kTOp + 32g) / lo [kTOp + 64 + 32g) (P is consumed)
      mbar_wait(bar(C_FULL), ph);
      tc_fence_after();
      if (warp == 8 && lane == 0) TL(lt, 4);
      {
        uint32_t c[32];
        tmem_ld32(lane_base + kTR + uint32_t(32 * g), c);
        st_split16<kTerms>(lane_base + kTOp + uint32_t(32 * g), 64u, c);
        st_split16<kTerms>(lane_base + kTOp + uint32_t(32 * g + 16), 64u, c + 16);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar(C_READY));
      // ---- Z columns [32g, 32g+32) -> global
      mbar_wait(bar(Z_FULL), ph);
      tc_fence_after();
      if (warp == 8 && lane == 0) TL(lt, 5);
      {
        uint32_t z[32];
        tmem_ld32(lane_base + kTR + 64u + uint32_t(32 * g), z);
        if (inst < p.batch && row < p.S) {
          float4* out = reinterpret_cast<float4*>(p.Z + int64_t(inst) * p.sZ + int64_t(row) * p.ldz + 32 * g);
#pragma unroll
          for (int j4 = 0; j4 < 8; ++j4)
            out[j4] = make_float4(__uint_as_float(z[4 * j4]), __uint_as_float(z[4 * j4 + 1]),
                                  __uint_as_float(z[4 * j4 + 2]), __uint_as_float(z[4 * j4 + 3]));
        }
      }
      tc_fence_before();
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
#if HS_DBG_TIMELINE
  if (blockIdx.x == 0)
    for (int i = threadIdx.x; i < 8 * 32; i += blockDim.x) g_head_timeline[i] = s_tl[i];
#endif
}

// 3-D fp32 tensor map with 64-byte swizzle (16-element boxes along the contiguous dim)
bool make_map_sw64(CUtensorMap* m, const void* ptr, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1, uint64_t s2,
                   uint32_t b0, uint32_t b1) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {s1, s2};
  cuuint32_t box[3] = {b0, b1, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(ptr), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

}  // namespace hs

// timing experiment only: reset / copy the debug timeline (8 x 32 slots)
extern "C" int hs_debug_head_timeline_reset(void) {
#if HS_DBG_TIMELINE
  static const long long zeros[256] = {};
  return cudaMemcpyToSymbol(hs::g_head_timeline, zeros, sizeof(zeros)) == cudaSuccess ? 0 : 1;
#else
  return 1;
#endif
}
extern "C" int hs_debug_head_timeline(long long* out) {
#if HS_DBG_TIMELINE
  return cudaMemcpyFromSymbol(out, hs::g_head_timeline, sizeof(long long) * 256) == cudaSuccess ? 0 : 1;
#else
  (void)out;
  return 1;
#endif
}

namespace hs {

bool head_fused_supported(const HeadArgs& a) {
  if (a.S < 1 || a.S > kS || a.dk != kDK || a.D < kWK || a.D % kWK || a.batch < 1 || !a.Wqkv || !a.Wh) return false;
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  if (!al16(a.X) || !al16(a.Z) || !al16(a.Wqkv) || !al16(a.Wh)) return false;
  const int64_t ld = a.ldz ? a.ldz : kDK;
  if ((a.sX | a.sZ | ld) & 3) return false;
  return tc::encode_fn() != nullptr;
}

cudaError_t head_fused(const HeadArgs& a, int terms, cudaStream_t s) {
  if (!head_fused_supported(a)) return cudaErrorInvalidValue;
  auto kernel = terms > 1 ? head_kernel<3> : head_kernel<1>;
  static std::once_flag once3, once1;
  static cudaError_t err3 = cudaSuccess, err1 = cudaSuccess;
  std::call_once(terms > 1 ? once3 : once1, [&] {
    (terms > 1 ? err3 : err1) = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
  });
  if (cudaError_t e = terms > 1 ? err3 : err1) return e;
  const uint64_t S = uint64_t(a.S), D = uint64_t(a.D), B = uint64_t(a.batch);
  CUtensorMap mX, mW, mWh, mXp;
  const bool ok = (kXK == 32 ? tc::make_map(&mX, a.X, D, S, B, D * 4, uint64_t(a.sX ? a.sX : S * D) * 4, kXK, kS, true)
                              : make_map_sw64(&mX, a.X, D, S, B, D * 4, uint64_t(a.sX ? a.sX : S * D) * 4, kXK, kS)) &&
                  tc::make_map(&mXp, a.X, D, S, B, D * 4, uint64_t(a.sX ? a.sX : S * D) * 4, kWK, kS, true) &&
                  (kWK == 32 ? tc::make_map(&mW, a.Wqkv, D, kN, 2, D * 4, uint64_t(kN) * D * 4, kWK, kN / 2, true)
                             : make_map_sw64(&mW, a.Wqkv, D, kN, 2, D * 4, uint64_t(kN) * D * 4, kWK, kN / 2)) &&
                  tc::make_map(&mWh, a.Wh, kDK, kDK, 2, kDK * 4, uint64_t(kDK * kDK) * 4, 32, kDK, true);
  if (!ok) return cudaErrorInvalidValue;
  const int64_t ldz = a.ldz ? a.ldz : kDK;
  HeadParams p{a.S, a.D, a.batch, (a.batch + 1) / 2, a.scale, a.Z, a.sZ ? a.sZ : int64_t(S) * ldz, ldz};
  const int max_pairs = tc::num_sms() / 2;
  const int pairs = p.pairs < max_pairs ? p.pairs : max_pairs;
  return launch_node(kernel, dim3(2 * pairs), dim3(kThreads), kSmem, s, 2, mX, mW, mWh, mXp, p);
}

}  // namespace hs
