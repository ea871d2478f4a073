// tcgen05 / TMEM / TMA GEMM for sm_100a with an fp32-accurate 3xTF32 mode.
//
//   C[M,N] (+ReLU) = A[M,K] · B        B = [K,N] row-major (nn) or [N,K] (nt)
//
// Persistent kernel: one CTA per SM walks the 128 x BN output tiles of all
// `batch` instances (instance index fastest, so concurrently running CTAs
// share the same weight tile in L2). Warp roles (512 threads):
//   warp 0       TMA producer. A (fp32) -> staging ring (SWIZZLE_128B); B either
//                as fp32 staging (activations) or, for resident weights, as
//                pre-split tf32 hi/lo planes (SW128, the canonical K-major UMMA
//                layout) written straight into the shared-memory operand ring.
//   warp 1       MMA issuer (one lane): tcgen05.mma.kind::tf32, accumulator in
//                TMEM, double-buffered (2 x BN columns) so the epilogue of tile
//                i overlaps the main loop of tile i+1.
//   warp 2       TMEM allocator.
//   warps 4..7   epilogue: tcgen05.ld 32x32b -> ReLU -> global (TMEM lane
//                quarter = warp % 4).
//   warps 8..15  converters: x = hi + lo with hi = cvt.rna.tf32(x), lo = x - hi
//                (exact). The split A goes to TMEM (tcgen05.st; the MMA reads A
//                from TMEM), so shared memory only carries B: this is what keeps
//                the kernel off the shared-memory bandwidth ceiling. Activation
//                B is split into shared memory (transposed when it is [K,N]).
// 3xTF32: D += Alo·Bhi + Ahi·Blo + Ahi·Bhi (Alo·Blo, ~2^-22 relative, is
// dropped). TF32 mode (terms = 1) issues only Ahi·Bhi.
//
// mbarrier pipelines: staging full/empty (TMA <-> converters), operand
// full/empty (converters + TMA <-> MMA, released by tcgen05.commit),
// accumulator full/empty (MMA <-> epilogue). TMA zero-fills out-of-bounds
// boxes, so ragged M/N/K need no special casing in the main loop.
#include <cuda.h>
#include <cuda_runtime.h>

#include <mutex>

#include "kernels.cuh"
#include "launch.cuh"
#include "tc_common.cuh"

namespace hs {

#ifndef HS_DBG_GEMM_TL  // timing experiment only: clock64 stamps of CTA 0 of gemm_tc_kernel
#define HS_DBG_GEMM_TL 0
#endif
#if HS_DBG_GEMM_TL
__device__ long long g_gemm_tl[16];
#define GTL(k)                                                                  \
  do {                                                                          \
    if (blockIdx.x == 0 && g_gemm_tl[k] == 0) g_gemm_tl[k] = clock64();         \
  } while (0)
#else
#define GTL(k) \
  do {         \
  } while (0)
#endif

namespace {

using namespace tc;

#ifndef HS_SMEM_BUDGET_KB
#define HS_SMEM_BUDGET_KB 200
#endif
#ifndef HS_NO_CAP
#define HS_NO_CAP 4  // max TMEM A stages
#endif
// Timing experiments only (profiles/): skip data movement / A conversion.
#ifndef HS_DBG_NOTMA
#define HS_DBG_NOTMA 0
#endif
#ifndef HS_DBG_NOCONV
#define HS_DBG_NOCONV 0
#endif
#ifndef HS_SMALL_GEMM
#define HS_SMALL_GEMM 1
#endif
#ifndef HS_DBG_NOEPI
#define HS_DBG_NOEPI 0
#endif
#ifndef HS_SPLIT_K  // split-K with red.global.add for latency-bound single-CTA launches
#define HS_SPLIT_K 1
#endif
#ifndef HS_CSPLIT_MAX  // cluster split-K: CTAs per cluster at most (0/1: red.add split-K only)
#define HS_CSPLIT_MAX 8
#endif
constexpr int kCsplitCap = HS_CSPLIT_MAX > 8 ? 16 : 8;  // partial registers per reducing thread
#ifndef HS_SPLIT_MIN_KB  // K-blocks per split at least
#define HS_SPLIT_MIN_KB 1
#endif
#ifndef HS_DBG_EARLYREL
#define HS_DBG_EARLYREL 0
#endif
constexpr int kEpiWarps = 4;
constexpr int kEpiTileBytes = 32 * 33 * 4;  // padded 32x32 fp32 transpose tile per epilogue warp
// Converters work in groups of 4 warps (one per TMEM lane quarter); group g
// handles the K-blocks with it % kConvGroups == g, so kConvGroups K-blocks are
// split concurrently and the per-block latency chain (smem load -> split ->
// tcgen05.st -> wait::st -> arrive) is overlapped instead of serialised.
// Stage counts are multiples of kConvGroups so each group revisits only its
// own slots, one phase at a time (a parity wait two phases ahead would alias).
#ifndef HS_CONV_GROUPS
#define HS_CONV_GROUPS 2
#endif
constexpr int kConvGroups = HS_CONV_GROUPS;
constexpr int kGroupWarps = 4;
constexpr int kConvWarps = kConvGroups * kGroupWarps;
constexpr int kThreads = 32 * (4 + kEpiWarps + kConvWarps);  // 4 control + 4 epilogue + converter warps
static_assert(kThreads <= 1024, "warp-role layout");


// B source: 0 = activation [N,K] (nt), 1 = activation [K,N] (nn), 2 = pre-split planes
// kSmall: configuration for short-K GEMMs (<= 4 K-blocks: attention QK^T,
// P·V, C·W_h). Two CTAs share an SM (256 TMEM columns, ~100 KB smem each), so
// the fixed prologue/epilogue latency of one tile overlaps another tile's work
// and kernels of concurrently running components can co-reside.
// kBf16: BF16x3 math (pre-split weights only): A and B split into bf16 hi/lo,
// D += Alo·Bhi + Ahi·Blo + Ahi·Bhi with kind::f16 MMAs (K=16 per instruction,
// twice the tf32 rate); B planes are 32 bf16 = 64-byte SW64 rows per K-block,
// A stages are 16 + 16 TMEM columns (bf16 pairs packed per 32-bit column).
template <int BN, int kBSrc, bool kSmall = false, bool kBf16 = false>
struct Cfg {
  static_assert(!kBf16 || kBSrc == 2, "bf16x3 is implemented for pre-split (resident) B only");
  static constexpr bool kBPre = kBSrc == 2;
  static constexpr int kCtasPerSm = kSmall ? 2 : 1;
  static constexpr int kTmemCols = kSmall ? 256 : 512;
  static constexpr int kStageA = BM * BK * 4;              // 16 KB fp32 A tile (SW128 via TMA)
  static constexpr int kStageB = kBPre ? 0 : BN * BK * 4;  // fp32 B staging (activations only)
  static constexpr int kStaging = kStageA + kStageB;
  static constexpr int kPlaneB = BN * (kBf16 ? 64 : 128);  // one SW128 tf32 / SW64 bf16 plane of B
  static constexpr int kOperand = 2 * kPlaneB;             // B hi + lo (A lives in TMEM)
  static constexpr int kAStage = kBf16 ? 32 : 64;          // TMEM columns per A stage (hi + lo)
  // TMEM: BN-wide fp32 accumulator(s) + kNO A stages of kAStage columns (one
  // row per lane). Double-buffer the accumulator only when that still leaves
  // room for 4 A stages; wider tiles trade epilogue overlap for pipeline depth.
  static constexpr int kAccBufs = (2 * BN + (kSmall ? 2 : 4) * kAStage <= kTmemCols) ? 2 : 1;
  static constexpr int kAccCols = kAccBufs * BN;
  static constexpr int kBudget = HS_SMEM_BUDGET_KB * 1024;  // + barriers/alignment stays under the 227 KB opt-in limit
  static constexpr int kNOtm = (kTmemCols - kAccCols) / kAStage;
  static constexpr int kNOsm = (kBudget - 2 * kStaging) / kOperand;
  static constexpr int kNOmin = kNOtm < kNOsm ? kNOtm : kNOsm;
  static constexpr int kNOcap = kSmall ? 2 : (kNOmin < HS_NO_CAP ? kNOmin : HS_NO_CAP);
  static constexpr int kNO = kNOcap - kNOcap % kConvGroups;
  static constexpr int kNSraw = (kBudget - kNO * kOperand) / kStaging;
  static constexpr int kNScap = kSmall ? 2 : (kNSraw > 6 ? 6 : kNSraw);
  static constexpr int kNS = kNScap - kNScap % kConvGroups;
  static_assert(kAccCols + kNO * kAStage <= kTmemCols, "TMEM budget exceeded");
  static_assert(kNS % kConvGroups == 0 && kNO % kConvGroups == 0, "stage rings must divide among groups");
  static constexpr int kTotal =
      kNS * kStaging + kNO * kOperand + 1024 /*barriers*/ + kEpiWarps * kEpiTileBytes + 1024 /*align*/;
  // cluster split-K: the partial tile (128 rows, BN + 4 floats apart) fits the staging
  // and operand rings (both idle once the tile's last MMA has completed)
  static constexpr int kRedLd = BN + 4;
  static constexpr int kRedTile = BM * kRedLd * 4;  // one CTA's partial tile (bytes)
  // its own partial + the (S - 1) row slices the peers push to it (at most 15/16 of a tile)
  static constexpr bool kCsplitOk = kNS * kStaging + kNO * kOperand >= kRedTile + kRedTile / 16 * 15;
  static_assert(kNS >= 2 && kNO >= 2, "pipeline too shallow");
  static_assert(kTotal * kCtasPerSm <= 227 * 1024, "shared memory budget exceeded");
};

struct TileParams {
  float* C;
  int64_t sC;
  int M, N, K;
  int batch;
  int a_batched, b_batched;
  int relu;
  int m_tiles, n_tiles;
  int total_tiles;
  // Grouped launch (n_out > 0): N = n_out * Nm columns, member m owns columns
  // [m*Nm, (m+1)*Nm) and writes its own output Cs[m] (row stride Nm).
  int n_out, Nm;
  float* Cs[4];
  int64_t sCs[4];
  int64_t ldc;  // row stride of C (0 = N, or Nm for grouped launches)
  // Softmax epilogue (one tile covers all N columns): C = softmax_row(acc * escale).
  int softmax;
  float escale;
  // Split-K (single-CTA kernel, latency-bound launches): tile t computes output
  // tile t % base_tiles over K-block range split t / base_tiles and adds it into
  // C (zeroed before the launch) with red.global.add; total_tiles = base * split.
  int split_k, base_tiles;
  // Cluster split-K (csplit > 1, replaces the red.add split): the csplit CTAs of a
  // cluster compute K-block ranges of one output tile (split = cluster rank), leave
  // their partial accumulators in shared memory, and reduce them over DSMEM in rank
  // order (deterministic; no zeroed C, so no memset node before the launch); the
  // ReLU epilogue applies after the reduction.
  int csplit;
};


// A converter step: this thread's row of a 128 x 32 fp32 staging tile (K-major,
// SWIZZLE_128B) -> hi/lo split written to the TMEM A stage at `ta` (its lane
// quarter): tf32 hi -> columns [0,32), lo -> [32,64); bf16 hi/lo packed in
// pairs (lower k in the low half) -> [0,16) and [16,32).
template <int kTerms, bool kBf16>
__device__ __forceinline__ void split_a_to_tmem(uint32_t sa, uint32_t ta, int row) {
  if constexpr (kBf16) {
    // 32 fp32 of this row -> bf16 hi/lo, packed in pairs (lower k in the low half):
    // hi -> columns [0,16), lo -> [16,32) of the stage.
    uint32_t hi[16], lo[16];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      float4 x = lds128(sa + sw128(row, c));
      const uint32_t h01 = pack_bf16x2(x.x, x.y), h23 = pack_bf16x2(x.z, x.w);
      hi[2 * c] = h01;
      hi[2 * c + 1] = h23;
      lo[2 * c] = pack_bf16x2(x.x - __uint_as_float(h01 << 16), x.y - __uint_as_float(h01 & 0xFFFF0000u));
      lo[2 * c + 1] = pack_bf16x2(x.z - __uint_as_float(h23 << 16), x.w - __uint_as_float(h23 & 0xFFFF0000u));
    }
    if (!HS_DBG_NOCONV) {
      tmem_st16(ta, hi);
      tmem_st16(ta + 16u, lo);
    }
  } else
#pragma unroll
  for (int hh = 0; hh < (HS_DBG_NOCONV ? 0 : 2); ++hh) {
    uint32_t hi[16], lo[16];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      float4 x = lds128(sa + sw128(row, 4 * hh + c));
      const float xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float hv = tf32_rna(xs[e]);
        hi[4 * c + e] = __float_as_uint(hv);
        lo[4 * c + e] = __float_as_uint(tf32_lo(xs[e], hv));
      }
    }
    tmem_st16(ta + uint32_t(16 * hh), hi);
    if constexpr (kTerms > 1) tmem_st16(ta + 32u + uint32_t(16 * hh), lo);
  }
}

// Epilogue store of one 32-column chunk: v = this thread's row values for
// columns [c0, c0+32) of the tile; transposed through the warp's padded smem
// tile so each group of 8 lanes writes one full 128-byte row (coalesced).
// Rows >= M (or the whole chunk when !rows_valid) are not stored.
__device__ __forceinline__ void epi_store_chunk(const TileParams& p, uint32_t tile, const float (&v)[32], int lane,
                                                int q, int m0, int inst, int c0, bool rows_valid) {
  // destination of this 32-column chunk: the single C, or member m's C;
  // `ncols` valid columns, rows `ld` elements apart
  int ncols = p.N;
  float* cbase;
  if (p.n_out > 0) {
    const int m = c0 / p.Nm;
    c0 -= m * p.Nm;
    ncols = p.Nm;
    cbase = p.Cs[m] + int64_t(inst) * p.sCs[m];
  } else {
    cbase = p.C + int64_t(inst) * p.sC;
  }
  const int64_t ld = p.ldc ? p.ldc : ncols;
  // Latency-bound launches (one instance): each thread stores its own row's 32
  // columns straight from registers (8 x 16 B, or red.add for a K split) instead of
  // the coalescing transpose through shared memory, which costs ~2k cycles per tile.
  if (p.batch == 1 && !HS_DBG_NOEPI) {
    const int grow = m0 + q * 32 + lane;
    float* dst = cbase + int64_t(grow) * ld + c0;
    // warp-uniform choice (the transpose path below synchronises the warp)
    if (__all_sync(0xffffffffu, c0 + 32 <= ncols && (reinterpret_cast<uintptr_t>(dst) & 15u) == 0)) {
      if (rows_valid && grow < p.M) {
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) {
          if (p.split_k > 1)
            asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst + 4 * j4), "f"(v[4 * j4]),
                         "f"(v[4 * j4 + 1]), "f"(v[4 * j4 + 2]), "f"(v[4 * j4 + 3])
                         : "memory");
          else
            *reinterpret_cast<float4*>(dst + 4 * j4) =
                make_float4(v[4 * j4], v[4 * j4 + 1], v[4 * j4 + 2], v[4 * j4 + 3]);
        }
      }
      return;
    }
  }
#pragma unroll
  for (int j = 0; j < 32; ++j) sts32(tile + uint32_t(lane * 33 + j) * 4u, v[j]);
  __syncwarp();
  const int cq = (lane & 7) * 4, rsub = lane >> 3;
  const bool vec = c0 + 32 <= ncols && (ld & 3) == 0;
#pragma unroll
  for (int pass = 0; pass < 8; ++pass) {
    const int rr = pass * 4 + rsub;
    const int grow = m0 + q * 32 + rr;
    const uint32_t src = tile + uint32_t(rr * 33 + cq) * 4u;
    const float4 x = make_float4(lds32(src), lds32(src + 4), lds32(src + 8), lds32(src + 12));
    if (rows_valid && grow < p.M && !HS_DBG_NOEPI) {
      float* dst = cbase + int64_t(grow) * ld + c0 + cq;
      if (p.split_k > 1) {  // partial sum of a K split: accumulate into C
        if (vec) {
          asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(x.x), "f"(x.y), "f"(x.z),
                       "f"(x.w)
                       : "memory");
        } else {
          const float e[4] = {x.x, x.y, x.z, x.w};
          for (int i = 0; i < 4; ++i)
            if (c0 + cq + i < ncols) atomicAdd(dst + i, e[i]);
        }
      } else if (vec) {
        *reinterpret_cast<float4*>(dst) = x;
      } else {
        const float e[4] = {x.x, x.y, x.z, x.w};
        for (int i = 0; i < 4; ++i)
          if (c0 + cq + i < ncols) dst[i] = e[i];
      }
    }
  }
  __syncwarp();  // the next chunk reuses the tile
}

template <int BN, int kBSrc, int kTerms, bool kSmall, bool kBf16>
__global__ void __launch_bounds__(kThreads, kSmall ? 2 : 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, TileParams p) {
  using L = Cfg<BN, kBSrc, kSmall, kBf16>;
  constexpr int NS = L::kNS, NO = L::kNO, kRedLd = L::kRedLd;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t staging = base;
  const uint32_t operand = staging + NS * L::kStaging;
  const uint32_t bars = operand + NO * L::kOperand;
  auto st_full = [&](int s) { return bars + 8u * uint32_t(s); };
  auto st_empty = [&](int s) { return bars + 8u * uint32_t(NS + s); };
  auto op_full = [&](int s) { return bars + 8u * uint32_t(2 * NS + s); };
  auto op_empty = [&](int s) { return bars + 8u * uint32_t(2 * NS + NO + s); };
  auto acc_full = [&](int a) { return bars + 8u * uint32_t(2 * NS + 2 * NO + a); };
  auto acc_empty = [&](int a) { return bars + 8u * uint32_t(2 * NS + 2 * NO + 2 + a); };
  const uint32_t tmem_slot = bars + 8u * uint32_t(2 * NS + 2 * NO + 4);
  const uint32_t red_full = bars + 8u * uint32_t(2 * NS + 2 * NO + 5);  // cluster split-K: peers' slices landed
  const uint32_t scratch = bars + 1024u;  // epilogue transpose tiles, one per epilogue warp
  const uint32_t* tmem_slot_ptr = reinterpret_cast<const uint32_t*>(smem_raw + (tmem_slot - smem_u32(smem_raw)));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) GTL(0);
  const int nk = (p.K + BK - 1) / BK;
  // K-block range of tile t (the whole K unless split-K)
  auto kb_begin = [&](int t) { return (t / p.base_tiles) * nk / p.split_k; };
  auto kb_end = [&](int t) { return (t / p.base_tiles + 1) * nk / p.split_k; };
  // first tile and stride of this CTA's persistent loop (cluster split-K: exactly one
  // tile, split = cluster rank, output tile = cluster index)
  const bool csplit = p.csplit > 1;
  const int t0 = csplit ? int(cluster_ctarank()) * p.base_tiles + int(blockIdx.x) / p.csplit : int(blockIdx.x);
  const int tstep = csplit ? p.total_tiles : int(gridDim.x);

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(st_full(s), 1);
      mbar_init(st_empty(s), kGroupWarps);
    }
    for (int s = 0; s < NO; ++s) {
      mbar_init(op_full(s), kGroupWarps + (L::kBPre ? 1 : 0));
      mbar_init(op_empty(s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(acc_full(a), 1);
      mbar_init(acc_empty(a), kEpiWarps);
    }
    mbar_init(red_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tmem_slot),
                 "r"(L::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  if (threadIdx.x == 0) GTL(1);
  pdl_launch_dependents();  // PDL (launch.cuh): the prologue above overlaps the previous kernel
  pdl_wait();
  if (threadIdx.x == 0) GTL(2);
  const uint32_t tmem = *tmem_slot_ptr;
  const uint32_t tmem_a = tmem + uint32_t(L::kAccCols);  // A stages start after the accumulators

  // tile index -> (m_tile, instance, n_tile); instance fastest after m.
  auto decode = [&](int t, int& m0, int& inst, int& n0) {
    t %= p.base_tiles;
    const int mt = t % p.m_tiles;
    const int rest = t / p.m_tiles;
    inst = rest % p.batch;
    n0 = (rest / p.batch) * BN;
    m0 = mt * BM;
  };

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      uint32_t it = 0;
      for (int t = t0; t < p.total_tiles; t += tstep) {
        int m0, inst, n0;
        decode(t, m0, inst, n0);
        const int ia = p.a_batched ? inst : 0, ib = p.b_batched ? inst : 0;
        for (int kb = kb_begin(t); kb < kb_end(t); ++kb, ++it) {
          const int s = int(it % NS);
          mbar_wait(st_empty(s), ((it / NS) & 1u) ^ 1u);
          const uint32_t sa = staging + uint32_t(s) * L::kStaging;
#if HS_DBG_NOTMA  // timing experiment only: no data movement
          mbar_arrive(st_full(s));
          (void)sa; (void)ia; (void)ib; (void)m0;
#else
          mbar_expect_tx(st_full(s), L::kStaging);
          GTL(3);
          tma_load_3d(sa, &tmA, st_full(s), kb * BK, m0, ia);
          if constexpr (kBSrc == 0) tma_load_3d(sa + L::kStageA, &tmB, st_full(s), kb * BK, n0, ib);
          if constexpr (kBSrc == 1) tma_load_3d(sa + L::kStageA, &tmB, st_full(s), n0, kb * BK, ib);
#endif
        }
      }
    }
  } else if (warp == 3) {
    // ------------------------------------------------------------ weight producer
    // Pre-split weight planes (hi at plane 0, lo at plane 1) straight into the
    // operand ring. A separate thread from the A producer, so A prefetch runs
    // kNS deep instead of stalling behind the operand ring.
    if constexpr (L::kBPre) {
      if (lane == 0) {
        uint32_t it = 0;
        for (int t = t0; t < p.total_tiles; t += tstep) {
          int m0, inst, n0;
          decode(t, m0, inst, n0);
          for (int kb = kb_begin(t); kb < kb_end(t); ++kb, ++it) {
            const int o = int(it % NO);
            mbar_wait(op_empty(o), ((it / NO) & 1u) ^ 1u);
            const uint32_t b_hi = operand + uint32_t(o) * L::kOperand;
#if HS_DBG_NOTMA
            mbar_arrive(op_full(o));
            (void)b_hi;
#else
            mbar_expect_tx(op_full(o), (kTerms > 1 ? 2 : 1) * L::kPlaneB);
            tma_load_3d(b_hi, &tmB, op_full(o), kb * BK, n0, 0);
            if constexpr (kTerms > 1) tma_load_3d(b_hi + L::kPlaneB, &tmB, op_full(o), kb * BK, n0, 1);
#endif
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = kBf16 ? instr_desc_bf16(BN) : instr_desc_tf32(BN);
      uint32_t it = 0, lt = 0;
      for (int t = t0; t < p.total_tiles; t += tstep, ++lt) {
        const uint32_t acc = lt % uint32_t(L::kAccBufs);
        mbar_wait(acc_empty(int(acc)), ((lt / uint32_t(L::kAccBufs)) & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t d = tmem + acc * uint32_t(BN);
        const int kb0 = kb_begin(t);
        for (int kb = kb0; kb < kb_end(t); ++kb, ++it) {
          const int o = int(it % NO);
          mbar_wait(op_full(o), (it / NO) & 1u);
          tc_fence_after();
          const uint32_t a_hi = tmem_a + uint32_t(o) * uint32_t(L::kAStage);
          const uint32_t a_lo = a_hi + uint32_t(L::kAStage / 2);
          const uint32_t b_hi = operand + uint32_t(o) * L::kOperand;
          const uint32_t b_lo = b_hi + L::kPlaneB;
          if constexpr (kBf16) {
            // K = 16 bf16 per instruction: 8 TMEM columns of packed pairs, 32 bytes of a SW64 row
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              const uint32_t kcol = uint32_t(kk) * 8u, koff = uint32_t(kk) * 32u;
              const uint32_t first = ((kb - kb0) | kk) ? 1u : 0u;
              mma_f16_ts(d, a_lo + kcol, smem_desc_sw64(b_hi + koff), idesc, first);
              mma_f16_ts(d, a_hi + kcol, smem_desc_sw64(b_lo + koff), idesc, 1u);
              mma_f16_ts(d, a_hi + kcol, smem_desc_sw64(b_hi + koff), idesc, 1u);
            }
          } else
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {  // K = 8 tf32 per instruction
            const uint32_t kcol = uint32_t(kk) * 8u, koff = uint32_t(kk) * 32u;
            const uint32_t first = ((kb - kb0) | kk) ? 1u : 0u;
            if constexpr (kTerms > 1) {
              mma_tf32_ts(d, a_lo + kcol, smem_desc(b_hi + koff), idesc, first);
              mma_tf32_ts(d, a_hi + kcol, smem_desc(b_lo + koff), idesc, 1u);
              mma_tf32_ts(d, a_hi + kcol, smem_desc(b_hi + koff), idesc, 1u);
            } else {
              mma_tf32_ts(d, a_hi + kcol, smem_desc(b_hi + koff), idesc, first);
            }
          }
          mma_commit(op_empty(o));  // operand slot (TMEM A + smem B) free once these MMAs have read it
          GTL(6);
        }
        mma_commit(acc_full(int(acc)));
      }
    }
  } else if (warp >= 4 && warp < 4 + kEpiWarps) {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;  // TMEM lane quarter accessible to this warp
    uint32_t lt = 0;
    for (int t = t0; t < p.total_tiles; t += tstep, ++lt) {
      int m0, inst, n0;
      decode(t, m0, inst, n0);
      const uint32_t acc = lt % uint32_t(L::kAccBufs);
      mbar_wait(acc_full(int(acc)), (lt / uint32_t(L::kAccBufs)) & 1u);
      tc_fence_after();
      if (q == 0 && lane == 0) GTL(7);
      const uint32_t tacc = tmem + (uint32_t(q * 32) << 16) + acc * uint32_t(BN);
      // the partials overwrite A staging slots whose TMA writes (async proxy) were consumed
      if (csplit) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      // Softmax epilogue: this thread owns one full row of the tile (N <= BN).
      // Two read passes over TMEM give the row max and the sum of exp(s*x - max);
      // the store pass scales by 1/sum.
      // exp is ex2.approx on (s*x - max)*log2(e) (rel. error ~2^-21, far inside
      // the 1e-4 tolerance): one MUFU op instead of the ~20-instruction expf,
      // which matters because one warp per scheduler does all of this.
      float smax = 0.f, ssum = 1.f, sl = 0.f, ml = 0.f;
      if (p.softmax) {
        uint32_t r[32];
        smax = -INFINITY;
#pragma unroll 1
        for (int cb = 0; cb < BN / 32 && cb * 32 < p.N; ++cb) {
          tmem_ld32(tacc + uint32_t(cb * 32), r);
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (cb * 32 + j < p.N) smax = fmaxf(smax, __uint_as_float(r[j]) * p.escale);
        }
        sl = p.escale * 1.4426950408889634f;
        ml = smax * 1.4426950408889634f;
        // summation order: sequential over columns [0,64) and [64,128), then s0 + s1
        // (the fused attention head's order, attn_head.cu)
        float s2[2] = {0.f, 0.f};
#pragma unroll 1
        for (int cb = 0; cb < BN / 32 && cb * 32 < p.N; ++cb) {
          tmem_ld32(tacc + uint32_t(cb * 32), r);
          float acc_s = s2[cb >= 2];
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (cb * 32 + j < p.N) acc_s = acc_s + ex2_approx(fmaf(__uint_as_float(r[j]), sl, -ml));
          s2[cb >= 2] = acc_s;
        }
        ssum = 1.f / (s2[0] + s2[1]);  // used as the reciprocal below
      }
#pragma unroll 1
      for (int cb = 0; cb < BN / 32; ++cb) {
        uint32_t r[32];
        tmem_ld32(tacc + uint32_t(cb * 32), r);
        if (cb == BN / 32 - 1) {
          // accumulator drained into registers: hand it back to the MMA warp early
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(acc_empty(int(acc)));
        }
        if (csplit) {  // this split's partial row chunk -> own smem (reduced after the cluster barrier)
          const uint32_t dst = staging + uint32_t((q * 32 + lane) * kRedLd + cb * 32) * 4u;
#pragma unroll
          for (int j4 = 0; j4 < 8; ++j4)
            sts128(dst + uint32_t(j4) * 16u, make_float4(__uint_as_float(r[4 * j4]), __uint_as_float(r[4 * j4 + 1]),
                                                        __uint_as_float(r[4 * j4 + 2]), __uint_as_float(r[4 * j4 + 3])));
          continue;
        }
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          float x = __uint_as_float(r[j]);
          if (p.softmax) x = ex2_approx(fmaf(x, sl, -ml)) * ssum;
          v[j] = p.relu ? fmaxf(x, 0.f) : x;
        }
        epi_store_chunk(p, scratch + uint32_t(q) * uint32_t(kEpiTileBytes), v, lane, q, m0, inst, n0 + cb * 32, true);
      }
      if (q == 0 && lane == 0) GTL(8);
    }
  } else if (warp >= 8) {
    // ------------------------------------------------------------ converters
    // A: warp w of group g owns TMEM lane quarter w % 4 (rows 32q..32q+31);
    // each thread splits the 32 k-values of its row and writes them with
    // tcgen05.st (hi -> columns [0,32), lo -> [32,64) of the stage).
    const int g = (warp - 8) / kGroupWarps;
    const int t = threadIdx.x - 256 - g * kGroupWarps * 32;  // 0..127 within the group (B conversion index)
    constexpr int kCT = kGroupWarps * 32;
    const int q = warp & 3;
    const int row = q * 32 + lane;
    uint32_t it = 0;
    for (int tile = t0; tile < p.total_tiles; tile += tstep) {
      for (int kb = kb_begin(tile); kb < kb_end(tile); ++kb, ++it) {
        if (int(it % kConvGroups) != g) continue;
        const int s = int(it % NS), o = int(it % NO);
        mbar_wait(st_full(s), (it / NS) & 1u);
        if (q == 0 && lane == 0) GTL(4);
        mbar_wait(op_empty(o), ((it / NO) & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t sa = staging + uint32_t(s) * L::kStaging, sb = sa + L::kStageA;
        const uint32_t ta = tmem_a + (uint32_t(q * 32) << 16) + uint32_t(o) * uint32_t(L::kAStage);
        split_a_to_tmem<kTerms, kBf16>(sa, ta, row);
        const uint32_t b_hi = operand + uint32_t(o) * L::kOperand;
        const uint32_t b_lo = b_hi + L::kPlaneB;
        if constexpr (kBSrc == 0) {  // [N,K] staging (SW128) -> same offsets
#pragma unroll
          for (int j = 0; j < L::kStageB / 16 / kCT; ++j) {
            const uint32_t off = uint32_t(t + kCT * j) * 16u;
            split_store<kTerms>(b_hi, b_lo, off, lds128(sb + off));
          }
        } else if constexpr (kBSrc == 1) {
          // [32 k][BN n] staging (no swizzle): gather 4 consecutive k of one column
          // n (consecutive threads -> consecutive n: conflict-free), write one
          // 16-byte K-major chunk (8 rows x distinct chunks per quarter-warp).
#pragma unroll
          for (int j = 0; j < (BN * 8) / kCT; ++j) {
            const int id = t + kCT * j, n = id % BN, kc = id / BN;
            const uint32_t src = sb + uint32_t((kc * 4) * BN + n) * 4u;
            float4 x = make_float4(lds32(src), lds32(src + BN * 4), lds32(src + 2 * BN * 4), lds32(src + 3 * BN * 4));
            split_store<kTerms>(b_hi, b_lo, sw128(n, kc), x);
          }
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        if constexpr (!L::kBPre) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(st_empty(s));
          mbar_arrive(op_full(o));
          if (q == 0) GTL(5);
        }
      }
    }
  }
  if (threadIdx.x == 0) GTL(9);
  if (csplit) {
    // Every split's partial tile is in its CTA's smem ([128][BN + 4] at `staging`). CTA r
    // owns rows [r * 128 / S, (r + 1) * 128 / S): once every CTA of the cluster has its
    // partial written (cluster barrier; the receive areas reuse the rings the mainloop
    // has then finished with), each CTA pushes the row slice it holds for every peer into
    // that peer's receive area with one bulk DSMEM copy each (cp.async.bulk shared::cta ->
    // shared::cluster, completing on the peer's red_full), then sums its own rows over the
    // S slices in rank order (deterministic), applies the ReLU and stores them,
    // consecutive threads on consecutive columns (coalesced). A second cluster barrier
    // phase (arrived once a CTA's incoming slices have landed, waited before exit) keeps
    // every source slice alive until its copy is done. The barrier is .aligned: warps whose
    // roles looped in one lane reconverge first.
    const int S = p.csplit, rows = BM / S, rank = int(cluster_ctarank());
    const uint32_t slice = uint32_t(rows * kRedLd * 4);
    const uint32_t recv = staging + uint32_t(L::kRedTile);  // S - 1 slots, sender order
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // partials visible to the bulk copies
    __syncthreads();
    cluster_sync_all();
    if (threadIdx.x == 0) {
      GTL(11);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(red_full),
                   "r"(uint32_t(S - 1) * slice)
                   : "memory");
      for (int r = 0; r < S; ++r) {
        if (r == rank) continue;
        const uint32_t dst = recv + uint32_t(rank < r ? rank : rank - 1) * slice;
        asm volatile(
            "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                mapa_rank(dst, uint32_t(r))),
            "r"(staging + uint32_t(r) * slice), "r"(slice), "r"(mapa_rank(red_full, uint32_t(r)))
            : "memory");
      }
    }
    mbar_wait(red_full, 0);
    if (threadIdx.x == 0) GTL(12);
    __syncwarp();
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");  // phase 2: my slices landed
    int m0, inst, n0;
    decode(t0, m0, inst, n0);
    // destination of column c: the single C, or member c / Nm of a grouped launch
    const int64_t ld = p.ldc ? p.ldc : (p.n_out ? p.Nm : p.N);
    auto dst_of = [&](int grow, int gcol) {
      if (p.n_out == 0) return p.C + int64_t(inst) * p.sC + int64_t(grow) * ld + gcol;
      const int m = gcol / p.Nm;
      return p.Cs[m] + int64_t(inst) * p.sCs[m] + int64_t(grow) * ld + (gcol - m * p.Nm);
    };
    for (int id = int(threadIdx.x); id < rows * (BN / 4); id += kThreads) {
      const int lr = id / (BN / 4), c4 = (id % (BN / 4)) * 4;
      const uint32_t in_slice = uint32_t(lr * kRedLd + c4) * 4u;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int sp = 0; sp < kCsplitCap; ++sp) {
        if (sp >= S) break;
        const uint32_t a = sp == rank ? staging + uint32_t(rank) * slice + in_slice
                                      : recv + uint32_t(sp < rank ? sp : sp - 1) * slice + in_slice;
        const float4 x = lds128(a);
        if (sp == 0) {
          acc = x;
        } else {
          acc.x += x.x;
          acc.y += x.y;
          acc.z += x.z;
          acc.w += x.w;
        }
      }
      if (p.relu) acc = make_float4(fmaxf(acc.x, 0.f), fmaxf(acc.y, 0.f), fmaxf(acc.z, 0.f), fmaxf(acc.w, 0.f));
      const int grow = m0 + rank * rows + lr, gcol = n0 + c4;
      if (grow >= p.M || gcol >= p.N) continue;
      float* dst = dst_of(grow, gcol);
      if ((reinterpret_cast<uintptr_t>(dst) & 15u) == 0 && gcol + 4 <= p.N && (p.n_out == 0 || p.Nm % 4 == 0)) {
        *reinterpret_cast<float4*>(dst) = acc;
      } else {
        const float e[4] = {acc.x, acc.y, acc.z, acc.w};
        for (int i = 0; i < 4 && gcol + i < p.N; ++i) dst[i] = e[i];
      }
    }
    if (threadIdx.x == 0) GTL(13);
    __syncwarp();
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");  // every copy everywhere done
    if (threadIdx.x == 0) GTL(14);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(L::kTmemCols));
    if (lane == 0) GTL(10);
  }
}

// ============================================================ CTA-pair kernel
// cta_group::2 variant for resident (pre-split) B: a cluster of two CTAs on
// one TPC computes a 256 x BN tile with M = 256 tcgen05.mma instructions
// issued by the leader (rank 0). Each CTA brings its own 128 rows of A (its
// "row block": one (instance, m-tile), so a pair covers two instances of the
// batch) as a hi/lo split in its own TMEM, and BN/2 of the B columns in its
// own shared memory; each CTA's TMEM receives its 128 rows x BN columns.
// Why: N = 256 per instruction amortises the TMEM A-operand read (64 B/cycle)
// over twice the columns of the single-CTA N = 128 tile, and splitting B
// across the pair halves the per-SM shared-memory traffic for B (TMA write +
// three MMA reads per K-block), which is what bounds a single CTA at N = 256.
//
// Synchronisation (all mbarriers live in each CTA's smem; "leader's X" is
// reached through mapa + mbarrier.arrive.release.cluster):
//   st_full/st_empty   local: A TMA <-> converters (as the 1-CTA kernel)
//   op_full[o]         leader's only: both CTAs' converter warps arrive after
//                      their A stage is in TMEM; the leader's B producer posts
//                      expect_tx for both B halves; both halves' TMA (with
//                      .cta_group::2) complete_tx on it.
//   op_empty[o]        each CTA: tcgen05.commit multicast (mask 0b11)
//   acc_full[a]        each CTA: commit multicast at the end of a tile
//   acc_empty[a]       leader's only: both CTAs' epilogue warps arrive.
#ifndef HS_PAIR_NO_CAP
#define HS_PAIR_NO_CAP 4
#endif
#ifndef HS_PAIR_GEMM
#define HS_PAIR_GEMM 1
#endif
#ifndef HS_PAIR_BN  // pair tile width for N >= 256
#define HS_PAIR_BN 256
#endif
#ifndef HS_PAIR_DBL192  // 192-wide pair tiles keep two accumulators
#define HS_PAIR_DBL192 1
#endif
#ifndef HS_PAIR_WIDE_BN  // tile width of that route (two accumulators fit up to 192)
#define HS_PAIR_WIDE_BN 192
#endif
#ifndef HS_PAIR_WIDE_KMAX
#define HS_PAIR_WIDE_KMAX 1024
#endif
#ifndef HS_PAIR_WIDE_NMIN
#define HS_PAIR_WIDE_NMIN 1024
#endif
#ifndef HS_PAIR_WIDE192  // FFN1-shaped GEMMs on double-buffered 192-wide pair tiles
#define HS_PAIR_WIDE192 1
#endif
#ifndef HS_PAIR_PRESPLIT  // converters split the A tile into registers before waiting for the A stage
#define HS_PAIR_PRESPLIT 1
#endif
#ifndef HS_PAIR_RELAXED  // converters signal A stages with relaxed (not release) cluster arrives
#define HS_PAIR_RELAXED 1
#endif
// HS_PAIR_RZ: tcgen05 kind::tf32 truncates fp32 operands to tf32 (profiles/tf32_trunc_probe.cu),
// so the TMA-landed A tile is already the hi term of the split x = rz(x) + (x - rz(x)): the
// hi·B products read it from shared memory, and the converters write only
// lo = rna(x - rz(x)) to a 32-column TMEM stage (half the TMEM stores, no hi rounding). The
// staging slot is then released by the MMAs' commit instead of by the converters.
#ifndef HS_PAIR_RZ
#define HS_PAIR_RZ 0
#endif
#ifndef HS_PAIR_MIN_ASTAGES  // double-buffer the accumulator if this many A stages still fit
#define HS_PAIR_MIN_ASTAGES 4
#endif

template <int BN, bool kBf16>
struct CfgPair {
  static_assert(BN % 32 == 0 && BN <= 256, "pair tile N");
  static constexpr int kTmemCols = 512;
  static constexpr int kStaging = BM * BK * 4;                  // 16 KB fp32 A tile
  static constexpr int kHalfN = BN / 2;                          // B rows held by each CTA
  static constexpr int kPlaneB = kHalfN * (kBf16 ? 64 : 128);   // one SW128 tf32 / SW64 bf16 half plane
  static constexpr int kOperand = 2 * kPlaneB;
  static constexpr bool kRZ = HS_PAIR_RZ && !kBf16;
  static constexpr int kAStage = kBf16 || kRZ ? 32 : 64;
  // BN = 192 keeps two accumulators (384 columns) beside two A stages, so the
  // epilogue of one tile overlaps the next tile's MMAs; BN = 256 needs all of TMEM
  // for one accumulator and four A stages.
  static constexpr int kMinAStages = (BN == 192 && HS_PAIR_DBL192) ? 2 : HS_PAIR_MIN_ASTAGES;
  static constexpr int kAccBufs = (2 * BN + kMinAStages * kAStage <= kTmemCols) ? 2 : 1;
  static constexpr int kAccCols = kAccBufs * BN;
  static constexpr int kBudget = HS_SMEM_BUDGET_KB * 1024;
  static constexpr int kNOtm = (kTmemCols - kAccCols) / kAStage;
  static constexpr int kNOsm = (kBudget - 2 * kStaging) / kOperand;
  static constexpr int kNOmin = kNOtm < kNOsm ? kNOtm : kNOsm;
  static constexpr int kNOcap = kNOmin < HS_PAIR_NO_CAP ? kNOmin : HS_PAIR_NO_CAP;
  static constexpr int kNO = kNOcap - kNOcap % kConvGroups;
  static constexpr int kNSraw = (kBudget - kNO * kOperand) / kStaging;
  static constexpr int kNScap = kNSraw > 8 ? 8 : kNSraw;
  static constexpr int kNS = kNScap - kNScap % kConvGroups;
  static_assert(kAccCols + kNO * kAStage <= kTmemCols, "TMEM budget exceeded");
  static_assert(kNS >= 2 && kNO >= 2, "pipeline too shallow");
  // epilogue: per warp two 32 x 32 fp32 SW128 staging tiles for TMA stores
  static constexpr int kEpiStage = 32 * 32 * 4;
  static constexpr int kTotal = kNS * kStaging + kNO * kOperand + 1024 + kEpiWarps * 2 * kEpiStage + 1024;
  static_assert(kTotal <= 227 * 1024, "shared memory budget exceeded");
};

// Output tensor maps for TMA stores: one per output (member) matrix.
struct CMaps {
  CUtensorMap m[4];
};


template <int BN, int kTerms, bool kBf16>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CMaps tmC, TileParams p) {
  using L = CfgPair<BN, kBf16>;
  constexpr int NS = L::kNS, NO = L::kNO;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t staging = base;
  const uint32_t operand = staging + NS * L::kStaging;
  const uint32_t bars = operand + NO * L::kOperand;
  auto st_full = [&](int s) { return bars + 8u * uint32_t(s); };
  auto st_empty = [&](int s) { return bars + 8u * uint32_t(NS + s); };
  auto op_full = [&](int s) { return bars + 8u * uint32_t(2 * NS + s); };
  auto op_empty = [&](int s) { return bars + 8u * uint32_t(2 * NS + NO + s); };
  auto acc_full = [&](int a) { return bars + 8u * uint32_t(2 * NS + 2 * NO + a); };
  auto acc_empty = [&](int a) { return bars + 8u * uint32_t(2 * NS + 2 * NO + 2 + a); };
  const uint32_t tmem_slot = bars + 8u * uint32_t(2 * NS + 2 * NO + 4);
  const uint32_t scratch = bars + 1024u;
  const uint32_t* tmem_slot_ptr = reinterpret_cast<const uint32_t*>(smem_raw + (tmem_slot - smem_u32(smem_raw)));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nk = (p.K + BK - 1) / BK;
  const uint32_t rank = cluster_ctarank();
  const int pair0 = int(cluster_id_x()), npairs = int(nclusters_x());
  const int total_rb = p.batch * p.m_tiles;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(st_full(s), 1);
      mbar_init(st_empty(s), L::kRZ ? 1 : kGroupWarps);  // RZ: the leader's commit (multicast)
    }
    for (int s = 0; s < NO; ++s) {
      mbar_init(op_full(s), 2 * kGroupWarps + 1);
      mbar_init(op_empty(s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(acc_full(a), 1);
      mbar_init(acc_empty(a), 2 * kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tmem_slot),
                 "r"(L::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();  // barriers initialised and TMEM allocated in both CTAs
  tc_fence_after();
  pdl_launch_dependents();  // PDL (launch.cuh)
  pdl_wait();
  const uint32_t tmem = *tmem_slot_ptr;
  const uint32_t tmem_a = tmem + uint32_t(L::kAccCols);

  // pair tile t -> (n0, this CTA's row block rb = (instance, m-tile)); n fastest,
  // so the pairs running at once share A row blocks through L2.
  auto decode = [&](int t, int& n0, int& inst, int& m0, bool& valid) {
    const int nt = t % p.n_tiles, rp = t / p.n_tiles;
    const int rb = 2 * rp + int(rank);
    valid = rb < total_rb;
    inst = rb / p.m_tiles;
    m0 = (rb % p.m_tiles) * BM;
    n0 = nt * BN;
  };
  // Columns the tile's MMAs cover: BN, or for a ragged last tile its valid columns
  // rounded up to 64 (FFN1: N = 2048 = 10 x 192 + 128), so no MMA work or epilogue
  // drain is spent on padding. Each CTA holds half of them as its B rows.
  auto tile_n = [&](int n0) {
    const int valid = p.N - n0;
    return valid >= BN ? BN : ((valid + 63) / 64) * 64;
  };

  if (warp == 0) {
    // ------------------------------------------------------------ A producer (local)
    if (lane == 0) {
      uint32_t it = 0;
      for (int t = pair0; t < p.total_tiles; t += npairs) {
        int n0, inst, m0;
        bool valid;
        decode(t, n0, inst, m0, valid);
        const int ia = p.a_batched ? inst : 0;  // inst >= batch (odd tail) -> zero-filled box
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = int(it % NS);
          mbar_wait(st_empty(s), ((it / NS) & 1u) ^ 1u);
          const uint32_t sa = staging + uint32_t(s) * L::kStaging;
#if HS_DBG_NOTMA
          mbar_arrive(st_full(s));
          (void)sa; (void)ia; (void)m0;
#else
          mbar_expect_tx(st_full(s), L::kStaging);
          tma_load_3d(sa, &tmA, st_full(s), kb * BK, m0, ia);
#endif
        }
      }
    }
  } else if (warp == 3) {
    // ------------------------------------------------------------ B producer: this CTA's half
    if (lane == 0) {
      uint32_t it = 0;
      for (int t = pair0; t < p.total_tiles; t += npairs) {
        int n0, inst, m0;
        bool valid;
        decode(t, n0, inst, m0, valid);
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int o = int(it % NO);
          mbar_wait(op_empty(o), ((it / NO) & 1u) ^ 1u);
          const uint32_t b_hi = operand + uint32_t(o) * L::kOperand;
          const uint32_t full = mapa_rank(op_full(o), 0);
#if HS_DBG_NOTMA
          if (rank == 0) mbar_arrive(op_full(o));
          (void)b_hi; (void)full;
#else
          if (rank == 0) mbar_expect_tx(op_full(o), 2 * (kTerms > 1 ? 2 : 1) * L::kPlaneB);
          const int nrow = n0 + int(rank) * (tile_n(n0) / 2);
          tma_load_3d_pair(b_hi, &tmB, full, kb * BK, nrow, 0);
          if constexpr (kTerms > 1) tma_load_3d_pair(b_hi + L::kPlaneB, &tmB, full, kb * BK, nrow, 1);
#endif
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader only)
    if (lane == 0 && rank == 0) {
      constexpr uint32_t idesc_bn = (kBf16 ? instr_desc_bf16(BN) : instr_desc_tf32(BN)) + (uint32_t(BM >> 4) << 24);
      uint32_t it = 0, lt = 0;
      for (int t = pair0; t < p.total_tiles; t += npairs, ++lt) {
        const uint32_t acc = lt % uint32_t(L::kAccBufs);
        mbar_wait(acc_empty(int(acc)), ((lt / uint32_t(L::kAccBufs)) & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t d = tmem + acc * uint32_t(BN);
        const uint32_t idesc = (idesc_bn & ~(0x3Fu << 17)) | (uint32_t(tile_n((t % p.n_tiles) * BN) >> 3) << 17);
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int o = int(it % NO);
          mbar_wait(op_full(o), (it / NO) & 1u);
          tc_fence_after();
          const uint32_t a_hi = tmem_a + uint32_t(o) * uint32_t(L::kAStage);
          const uint32_t a_lo = a_hi + uint32_t(L::kAStage / 2);
          const uint32_t b_hi = operand + uint32_t(o) * L::kOperand;
          const uint32_t b_lo = b_hi + L::kPlaneB;
          if constexpr (kBf16) {
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              const uint32_t kcol = uint32_t(kk) * 8u, koff = uint32_t(kk) * 32u;
              const uint32_t first = (kb | kk) ? 1u : 0u;
              mma_pair_f16_ts(d, a_lo + kcol, smem_desc_sw64(b_hi + koff), idesc, first);
              mma_pair_f16_ts(d, a_hi + kcol, smem_desc_sw64(b_lo + koff), idesc, 1u);
              mma_pair_f16_ts(d, a_hi + kcol, smem_desc_sw64(b_hi + koff), idesc, 1u);
            }
          } else if constexpr (L::kRZ) {
            // lo·B_hi from the TMEM stage (lo at the stage's first 32 columns); hi·B_lo and
            // hi·B_hi read the raw A tile of staging slot s (each CTA its own 128 rows)
            const uint32_t sa = staging + uint32_t(it % NS) * L::kStaging;
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk) {
              const uint32_t kcol = uint32_t(kk) * 8u, koff = uint32_t(kk) * 32u;
              const uint32_t first = (kb | kk) ? 1u : 0u;
              const uint64_t ad = smem_desc(sa + koff);
              if constexpr (kTerms > 1) {
                mma_pair_tf32_ts(d, a_hi + kcol, smem_desc(b_hi + koff), idesc, first);
                mma_pair_tf32_ss(d, ad, smem_desc(b_lo + koff), idesc, 1u);
                mma_pair_tf32_ss(d, ad, smem_desc(b_hi + koff), idesc, 1u);
              } else {
                mma_pair_tf32_ss(d, ad, smem_desc(b_hi + koff), idesc, first);
              }
            }
            mma_commit_pair(st_empty(int(it % NS)));
          } else {
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk) {
              const uint32_t kcol = uint32_t(kk) * 8u, koff = uint32_t(kk) * 32u;
              const uint32_t first = (kb | kk) ? 1u : 0u;
              if constexpr (kTerms > 1) {
                mma_pair_tf32_ts(d, a_lo + kcol, smem_desc(b_hi + koff), idesc, first);
                mma_pair_tf32_ts(d, a_hi + kcol, smem_desc(b_lo + koff), idesc, 1u);
                mma_pair_tf32_ts(d, a_hi + kcol, smem_desc(b_hi + koff), idesc, 1u);
              } else {
                mma_pair_tf32_ts(d, a_hi + kcol, smem_desc(b_hi + koff), idesc, first);
              }
            }
          }
          mma_commit_pair(op_empty(o));
        }
        mma_commit_pair(acc_full(int(acc)));
      }
    }
  } else if (warp >= 4 && warp < 4 + kEpiWarps) {
    // ------------------------------------------------------------ epilogue (this CTA's rows)
    // TMEM -> registers -> (ReLU) -> SW128 smem staging tile -> TMA store. The
    // stores run asynchronously, so the accumulator is released as soon as its
    // last columns are in registers and the warps never wait on global writes.
    // Rows past M, columns past N and the odd row block of a ragged batch fall
    // outside the output tensor map and are clipped by the TMA unit.
    const int q = warp & 3;
    const uint32_t stage0 = scratch + uint32_t(q) * uint32_t(2 * L::kEpiStage);
    uint32_t lt = 0, cnt = 0;
    for (int t = pair0; t < p.total_tiles; t += npairs, ++lt) {
      int n0, inst, m0;
      bool valid;
      decode(t, n0, inst, m0, valid);
      const uint32_t acc = lt % uint32_t(L::kAccBufs);
      mbar_wait(acc_full(int(acc)), (lt / uint32_t(L::kAccBufs)) & 1u);
      tc_fence_after();
      const uint32_t tacc = tmem + (uint32_t(q * 32) << 16) + acc * uint32_t(BN);
#if HS_DBG_EARLYREL  // timing experiment only (wrong results): release the accumulator at once
      if (lane == 0) mbar_arrive_cluster(mapa_rank(acc_empty(int(acc)), 0));
#endif
      // one 32-column chunk: registers -> (ReLU) -> SW128 staging -> TMA store
      auto store_chunk = [&](const uint32_t (&r)[32], int cb) {
        int c0 = n0 + cb * 32;
        if (c0 >= p.N || !valid) return;
        int mi = 0;
        if (p.n_out > 0) {
          mi = c0 / p.Nm;
          c0 -= mi * p.Nm;
        }
        const uint32_t buf = stage0 + (cnt & 1u) * uint32_t(L::kEpiStage);
        if (cnt >= 2) {
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          __syncwarp();
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          float4 x = make_float4(__uint_as_float(r[4 * c]), __uint_as_float(r[4 * c + 1]),
                                 __uint_as_float(r[4 * c + 2]), __uint_as_float(r[4 * c + 3]));
          if (p.relu) x = make_float4(fmaxf(x.x, 0.f), fmaxf(x.y, 0.f), fmaxf(x.z, 0.f), fmaxf(x.w, 0.f));
          sts128(buf + uint32_t(lane) * 128u + (uint32_t(c ^ (lane & 7)) << 4), x);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0 && !HS_DBG_NOEPI) tma_store_3d(&tmC.m[mi], buf, c0, m0 + q * 32, inst);
        ++cnt;
      };
      // Two chunks per TMEM round trip (two tcgen05.ld in flight, one wait); the
      // accumulator is released as soon as the last pair is in registers.
      static_assert((BN / 32) % 2 == 0, "pair epilogue drains chunks in pairs");
#pragma unroll 1
      const int nchunks = tile_n(n0) / 32;
      for (int cb = 0; cb < nchunks; cb += 2) {
        uint32_t r0[32], r1[32];
        tmem_ld32_nowait(tacc + uint32_t(cb * 32), r0);
        tmem_ld32_nowait(tacc + uint32_t(cb * 32 + 32), r1);
        tmem_ld_wait(r0);
        tmem_ld_dep(r1);
        if (cb + 2 == nchunks && !HS_DBG_EARLYREL) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(mapa_rank(acc_empty(int(acc)), 0));
        }
        store_chunk(r0, cb);
        store_chunk(r1, cb + 1);
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  } else if (warp >= 8) {
    // ------------------------------------------------------------ converters (this CTA's A rows)
    const int g = (warp - 8) / kGroupWarps;
    const int q = warp & 3;
    const int row = q * 32 + lane;
    uint32_t it = 0;
    for (int tile = pair0; tile < p.total_tiles; tile += npairs) {
      for (int kb = 0; kb < nk; ++kb, ++it) {
        if (int(it % kConvGroups) != g) continue;
        const int s = int(it % NS), o = int(it % NO);
        mbar_wait(st_full(s), (it / NS) & 1u);
        const uint32_t sa = staging + uint32_t(s) * L::kStaging;
        const uint32_t ta = tmem_a + (uint32_t(q * 32) << 16) + uint32_t(o) * uint32_t(L::kAStage);
        bool staged_released = false;
        if constexpr (L::kRZ) {
          // lo = rna(x - rz(x)) of this row's 32 values -> the stage's 32 columns; the raw
          // tile stays in the staging slot for the MMAs (released by their commit)
          uint32_t lo[32];
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float4 x = lds128(sa + sw128(row, c));
            const float xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
            for (int e = 0; e < 4; ++e)
              lo[4 * c + e] = __float_as_uint(tf32_rna(xs[e] - __uint_as_float(__float_as_uint(xs[e]) & 0xFFFFE000u)));
          }
          staged_released = true;
          mbar_wait(op_empty(o), ((it / NO) & 1u) ^ 1u);
          tc_fence_after();
          if (kTerms > 1 && !HS_DBG_NOCONV) {
            tmem_st16(ta, *reinterpret_cast<const uint32_t(*)[16]>(lo));
            tmem_st16(ta + 16u, *reinterpret_cast<const uint32_t(*)[16]>(lo + 16));
          }
        } else if constexpr (!kBf16 && HS_PAIR_PRESPLIT) {
          // split this row's 32 values into registers and hand the staging tile back
          // before waiting for the A stage: only the TMEM stores remain between the
          // MMAs' release of the stage and its reuse (as in head_fused.cu)
          uint32_t hi[32], lo[32], dep = 0;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float4 x = lds128(sa + sw128(row, c));
            dep ^= __float_as_uint(x.x);  // one register of each LDS.128
            const float xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float hv = tf32_rna(xs[e]);
              hi[4 * c + e] = __float_as_uint(hv);
              lo[4 * c + e] = __float_as_uint(tf32_lo(xs[e], hv));
            }
          }
          // the slot goes back to TMA only once this warp's loads have returned
          if (lane == 0) mbar_arrive_after(st_empty(s), dep);
          staged_released = true;
          mbar_wait(op_empty(o), ((it / NO) & 1u) ^ 1u);
          tc_fence_after();
          if (!HS_DBG_NOCONV) {
            tmem_st16(ta, *reinterpret_cast<const uint32_t(*)[16]>(hi));
            tmem_st16(ta + 16u, *reinterpret_cast<const uint32_t(*)[16]>(hi + 16));
            if constexpr (kTerms > 1) {
              tmem_st16(ta + 32u, *reinterpret_cast<const uint32_t(*)[16]>(lo));
              tmem_st16(ta + 48u, *reinterpret_cast<const uint32_t(*)[16]>(lo + 16));
            }
          }
        } else {
          mbar_wait(op_empty(o), ((it / NO) & 1u) ^ 1u);
          tc_fence_after();
          split_a_to_tmem<kTerms, kBf16>(sa, ta, row);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (!staged_released) mbar_arrive(st_empty(s));
#if HS_PAIR_RELAXED
          // relaxed: the stage's TMEM stores are complete (tcgen05.wait::st above); a
          // release arrive at cluster scope costs ~1k cycles in this thread (head_fused.cu)
          asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(mapa_rank(op_full(o), 0))
                       : "memory");
#else
          mbar_arrive_cluster(mapa_rank(op_full(o), 0));
#endif
        }
      }
    }
  }
  tc_fence_before();
  cluster_sync_all();  // both CTAs done with TMEM, smem barriers and remote arrivals
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(L::kTmemCols));
  }
}

// Weight preparation: B (resident) -> K-major hi/lo planes [2][N][K], tf32
// (fp32 containers) or bf16 (hi = bf16_rn(x), lo = bf16_rn(x - hi)).
template <bool kNT>
__global__ void split_weights_bf16_kernel(const float* __restrict__ B, uint16_t* __restrict__ planes, int N, int K,
                                          int64_t plane) {
  __shared__ float tile[32][33];
  const int n0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    int n = n0 + (kNT ? i : threadIdx.x), k = k0 + (kNT ? threadIdx.x : i);
    float v = 0.f;
    if (n < N && k < K) v = kNT ? B[int64_t(n) * K + k] : B[int64_t(k) * N + n];
    if (kNT) tile[i][threadIdx.x] = v;
    else tile[threadIdx.x][i] = v;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    int n = n0 + i, k = k0 + threadIdx.x;
    if (n < N && k < K) {
      const float x = tile[i][threadIdx.x];
      const uint32_t h = pack_bf16x2(x, 0.f) & 0xFFFFu;
      const uint32_t l = pack_bf16x2(x - __uint_as_float(h << 16), 0.f) & 0xFFFFu;
      planes[int64_t(n) * K + k] = uint16_t(h);
      planes[plane + int64_t(n) * K + k] = uint16_t(l);
    }
  }
}

template <bool kNT>
__global__ void split_weights_kernel(const float* __restrict__ B, float* __restrict__ planes, int N, int K,
                                     int64_t plane) {
  __shared__ float tile[32][33];
  const int n0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    // load tile[n][k]
    int n = n0 + (kNT ? i : threadIdx.x), k = k0 + (kNT ? threadIdx.x : i);
    float v = 0.f;
    if (n < N && k < K) v = kNT ? B[int64_t(n) * K + k] : B[int64_t(k) * N + n];
    if (kNT) tile[i][threadIdx.x] = v;
    else tile[threadIdx.x][i] = v;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    int n = n0 + i, k = k0 + threadIdx.x;
    if (n < N && k < K) {
      float x = tile[i][threadIdx.x];
      float h = tf32_rna(x);
      planes[int64_t(n) * K + k] = h;
      planes[plane + int64_t(n) * K + k] = tf32_lo(x, h);
    }
  }
}

// ----------------------------------------------------------------- host side

template <int BN, int kBSrc, int kTerms, bool kSmall = false, bool kBf16 = false>
cudaError_t launch(const GemmArgs& a, cudaStream_t s) {
  using L = Cfg<BN, kBSrc, kSmall, kBf16>;
  auto kernel = gemm_tc_kernel<BN, kBSrc, kTerms, kSmall, kBf16>;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [&] {
    attr_err = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kTotal);
    // cluster split-K may use 16 CTAs per cluster (above the portable 8)
    if (attr_err == cudaSuccess && HS_CSPLIT_MAX > 8)
      attr_err = cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  });
  if (attr_err != cudaSuccess) return attr_err;
  const uint64_t M = uint64_t(a.M), N = uint64_t(a.N), K = uint64_t(a.K);
  const uint64_t nA = a.sA ? uint64_t(a.batch) : 1, nB = a.sB ? uint64_t(a.batch) : 1;
  const uint64_t sA = (a.sA ? uint64_t(a.sA) : M * K) * 4;
  CUtensorMap mA, mB;
  if (!make_map(&mA, a.A, K, M, nA, K * 4, sA, BK, BM, true)) return cudaErrorInvalidValue;
  bool ok = false;
  if constexpr (kBSrc == 2 && kBf16) {
    ok = make_map(&mB, a.Bplanes, K, N, 2, K * 2, N * K * 2, BK, BN, true, true);
  } else if constexpr (kBSrc == 2) {
    ok = make_map(&mB, a.Bplanes, K, N, 2, K * 4, N * K * 4, BK, BN, true);
  } else if constexpr (kBSrc == 0) {
    const uint64_t sB = (a.sB ? uint64_t(a.sB) : N * K) * 4;
    ok = make_map(&mB, a.B, K, N, nB, K * 4, sB, BK, BN, true);
  } else {
    const uint64_t sB = (a.sB ? uint64_t(a.sB) : N * K) * 4;
    ok = make_map(&mB, a.B, N, K, nB, N * 4, sB, BN, BK, false);
  }
  if (!ok) return cudaErrorInvalidValue;
  TileParams p{};
  p.C = a.C;
  p.sC = a.sC;
  p.M = a.M;
  p.N = a.N;
  p.K = a.K;
  p.batch = a.batch;
  p.a_batched = a.sA != 0;
  p.b_batched = a.sB != 0;
  p.relu = a.relu ? 1 : 0;
  p.m_tiles = (a.M + BM - 1) / BM;
  p.n_tiles = (a.N + BN - 1) / BN;
  p.n_out = a.n_out > 1 ? a.n_out : 0;
  p.Nm = p.n_out ? a.N / a.n_out : a.N;
  for (int i = 0; i < p.n_out; ++i) {
    p.Cs[i] = a.Cs[i];
    p.sCs[i] = a.sCs[i];
  }
  p.ldc = a.ldc;
  p.softmax = a.softmax;
  p.escale = a.escale;
  if (p.softmax && p.n_tiles != 1) return cudaErrorInvalidValue;
  const int base = p.m_tiles * p.n_tiles * a.batch;
  const int slots = num_sms() * L::kCtasPerSm;
  // Split-K for latency-bound single-instance launches (few output tiles, long K
  // loop: one instance's FFN2 runs 8 CTAs over 64 K-blocks). Preferred: cluster
  // split-K (p.csplit): S CTAs of a cluster split the K-blocks of one tile and
  // reduce their partials over DSMEM in rank order, so the result is deterministic,
  // ReLU applies after the sum, and C needs no zeroing (no memset node ahead of the
  // kernel). Otherwise (tiles whose partial does not fit the staging ring) each
  // split adds its partial into a zeroed C with red.global.add (not bit-
  // reproducible: fp32 addition order). Batched launches never split.
  const int nk = (a.K + BK - 1) / BK;
  int split = 1, csplit = 0;
  if (HS_SPLIT_K && a.batch == 1 && !a.softmax && nk >= 2 * HS_SPLIT_MIN_KB && 4 * base <= slots) {
    if constexpr (L::kCsplitOk) {
      if (HS_CSPLIT_MAX >= 2) {
        int S = slots / base;
        if (S > nk / HS_SPLIT_MIN_KB) S = nk / HS_SPLIT_MIN_KB;
        if (S > HS_CSPLIT_MAX) S = HS_CSPLIT_MAX;
        S = S >= 16 ? 16 : S >= 8 ? 8 : S >= 4 ? 4 : S >= 2 ? 2 : 1;  // rows of the reduction divide evenly
        if (S >= 2) split = csplit = S;
      }
    }
    if (!csplit && !a.deterministic && !a.relu && !a.ldc && p.n_out == 0) {
      split = slots / base;
      if (split > nk / HS_SPLIT_MIN_KB) split = nk / HS_SPLIT_MIN_KB;
      if (split > 16) split = 16;
      if (split < 2) split = 1;
    }
  }
  p.split_k = split;
  p.csplit = csplit;
  p.base_tiles = base;
  p.total_tiles = base * split;
  if (split > 1 && !csplit) {
    const cudaError_t e = cudaMemsetAsync(a.C, 0, size_t(a.batch) * size_t(a.M) * size_t(a.N) * 4, s);
    if (e != cudaSuccess) return e;
  }
  if (csplit) return launch_node(kernel, dim3(p.total_tiles), dim3(kThreads), L::kTotal, s, csplit, mA, mB, p);
  const int grid = p.total_tiles < slots ? p.total_tiles : slots;
  return launch_node(kernel, dim3(grid), dim3(kThreads), L::kTotal, s, 1, mA, mB, p);
}

// CTA-pair launch (resident B planes): clusters of 2, one pair per TPC,
// persistent over the 256 x BN pair tiles.
template <int BN, int kTerms, bool kBf16>
cudaError_t launch_pair(const GemmArgs& a, cudaStream_t s) {
  using L = CfgPair<BN, kBf16>;
  auto kernel = gemm_pair_kernel<BN, kTerms, kBf16>;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  static int max_pairs = 0;
  std::call_once(once, [&] {
    attr_err = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, L::kTotal);
    if (attr_err != cudaSuccess) return;
    cudaLaunchConfig_t q{};
    q.gridDim = dim3(2 * (num_sms() / 2));
    q.blockDim = dim3(kThreads);
    q.dynamicSmemBytes = L::kTotal;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    q.attrs = at;
    q.numAttrs = 1;
    int n = 0;
    attr_err = cudaOccupancyMaxActiveClusters(&n, kernel, &q);
    max_pairs = n > 0 ? n : num_sms() / 2;
  });
  if (attr_err != cudaSuccess) return attr_err;
  const uint64_t M = uint64_t(a.M), N = uint64_t(a.N), K = uint64_t(a.K);
  const uint64_t nA = a.sA ? uint64_t(a.batch) : 1;
  const uint64_t sA = (a.sA ? uint64_t(a.sA) : M * K) * 4;
  CUtensorMap mA, mB;
  if (!make_map(&mA, a.A, K, M, nA, K * 4, sA, BK, BM, true)) return cudaErrorInvalidValue;
  const uint64_t eb = kBf16 ? 2 : 4;
  if (!make_map(&mB, a.Bplanes, K, N, 2, K * eb, N * K * eb, BK, BN / 2, true, kBf16)) return cudaErrorInvalidValue;
  TileParams p{};
  p.C = a.C;
  p.sC = a.sC;
  p.M = a.M;
  p.N = a.N;
  p.K = a.K;
  p.batch = a.batch;
  p.a_batched = a.sA != 0;
  p.b_batched = 0;
  p.relu = a.relu ? 1 : 0;
  p.m_tiles = (a.M + BM - 1) / BM;
  p.n_tiles = (a.N + BN - 1) / BN;
  p.n_out = a.n_out > 1 ? a.n_out : 0;
  p.Nm = p.n_out ? a.N / a.n_out : a.N;
  for (int i = 0; i < p.n_out; ++i) {
    p.Cs[i] = a.Cs[i];
    p.sCs[i] = a.sCs[i];
  }
  p.ldc = a.ldc;
  // output maps: {columns, rows, instances}, 32 x 32 boxes, SW128 (matches the staging layout)
  CMaps mc{};
  const int nmaps = p.n_out ? p.n_out : 1;
  for (int i = 0; i < nmaps; ++i) {
    float* c = p.n_out ? a.Cs[i] : a.C;
    const uint64_t sc = uint64_t(p.n_out ? a.sCs[i] : a.sC);
    const uint64_t ncols = uint64_t(p.Nm);
    const uint64_t ld = a.ldc ? uint64_t(a.ldc) : ncols;
    if (!make_map(&mc.m[i], c, ncols, M, uint64_t(a.batch), ld * 4, (sc ? sc : ld * M) * 4, 32, 32, true))
      return cudaErrorInvalidValue;
  }
  const int row_pairs = (a.batch * p.m_tiles + 1) / 2;
  p.total_tiles = p.n_tiles * row_pairs;
  const int pairs = p.total_tiles < max_pairs ? p.total_tiles : max_pairs;
  return launch_node(kernel, dim3(2 * pairs), dim3(kThreads), L::kTotal, s, 2, mA, mB, mc, p);
}

template <int BN>
cudaError_t launch_pair_bn(const GemmArgs& a, int terms, cudaStream_t s) {
  if (a.bf16) return launch_pair<BN, 3, true>(a, s);
  return terms > 1 ? launch_pair<BN, 3, false>(a, s) : launch_pair<BN, 1, false>(a, s);
}

template <int BN, bool kSmall = false>
cudaError_t launch_bn(const GemmArgs& a, int terms, cudaStream_t s) {
  if (a.Bplanes && a.bf16) return launch<BN, 2, 3, kSmall, true>(a, s);
  if (a.Bplanes) return terms > 1 ? launch<BN, 2, 3, kSmall>(a, s) : launch<BN, 2, 1, kSmall>(a, s);
  if (a.layout == GemmLayout::nt) return terms > 1 ? launch<BN, 0, 3, kSmall>(a, s) : launch<BN, 0, 1, kSmall>(a, s);
  return terms > 1 ? launch<BN, 1, 3, kSmall>(a, s) : launch<BN, 1, 1, kSmall>(a, s);
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace

bool gemm_tcgen05_supported(const GemmArgs& a) {
  if (a.M < 1 || a.N < 1 || a.K < 1 || a.batch < 1) return false;
  if (a.K % 4 || (a.layout == GemmLayout::nn && !a.Bplanes && a.N % 4)) return false;
  if (a.sA % 4 || a.sB % 4 || a.sC % 4) return false;
  if (!aligned16(a.A) || !aligned16(a.B) || !aligned16(a.C)) return false;
  if (a.Bplanes && (!aligned16(a.Bplanes) || a.sB != 0)) return false;
  return encode_fn() != nullptr;
}

cudaError_t gemm_tcgen05(const GemmArgs& a, int terms, cudaStream_t s) {
  // Resident-weight GEMMs with wide N and at least two row blocks run on CTA
  // pairs (M = 256 tcgen05.mma over two instances / m-tiles).
  const int row_blocks = a.batch * ((a.M + BM - 1) / BM);
  bool store_ok = true;  // TMA stores: 16-byte aligned bases, row and instance strides
  const int nm = a.n_out > 1 ? a.n_out : 1;
  for (int i = 0; i < nm; ++i) {
    const void* c = a.n_out > 1 ? a.Cs[i] : a.C;
    const int64_t sc = a.n_out > 1 ? a.sCs[i] : a.sC;
    const int64_t ld = a.ldc ? a.ldc : (a.n_out > 1 ? a.N / a.n_out : a.N);
    if ((reinterpret_cast<uintptr_t>(c) & 15u) || (ld & 3) || (sc & 3) || (a.batch > 1 && sc == 0)) store_ok = false;
  }
  if (HS_PAIR_GEMM && store_ok && a.Bplanes && !a.softmax && row_blocks >= 2 &&
      !(a.n_out > 1 && a.N / a.n_out % 32)) {
    if (a.N == 192) return launch_pair_bn<192>(a, terms, s);
    // wide N over a short K (FFN1: N = 2048, K = 512): the per-tile epilogue drain is
    // ~10 % of a 256-wide tile's MMA time, so double-buffered 192-wide tiles win
    // despite the ragged last tile
    if (HS_PAIR_WIDE192 && a.n_out <= 1 && a.N >= HS_PAIR_WIDE_NMIN && a.K <= HS_PAIR_WIDE_KMAX)
      return launch_pair_bn<HS_PAIR_WIDE_BN>(a, terms, s);
    if (a.N >= 256 && a.n_out <= 1) return launch_pair_bn<HS_PAIR_BN>(a, terms, s);
  }
  if (a.n_out > 1) {
    // grouped launch: one tile covers every member (a.N = total columns)
    if (!a.Bplanes || a.N % a.n_out || (a.N / a.n_out) % 32 || a.n_out > 4) return cudaErrorInvalidValue;
    if (a.N == 128) return launch_bn<128>(a, terms, s);
    if (a.N == 192) {
      if (a.bf16) return launch<192, 2, 3, false, true>(a, s);
      return terms > 1 ? launch<192, 2, 3>(a, s) : launch<192, 2, 1>(a, s);
    }
    return cudaErrorInvalidValue;
  }
  // softmax epilogue: one 128-wide tile holds whole rows
  if (a.softmax) return a.N <= 128 ? launch_bn<128>(a, terms, s) : cudaErrorInvalidValue;
  // short K (attention-sized GEMMs): 64-wide tiles, two CTAs per SM
  if (a.K <= 4 * BK && a.N <= 128 && HS_SMALL_GEMM) return launch_bn<64, true>(a, terms, s);
  if (a.N <= 64) return launch_bn<64>(a, terms, s);
  // Latency-bound launches (a single instance's FFN, a 256^2 GEMM): when 128-wide
  // tiles would leave most SMs idle, 64-wide tiles halve each CTA's serial K loop
  // and double the CTAs working on it.
  const int tiles128 = row_blocks * ((a.N + 127) / 128);
  if (2 * tiles128 <= num_sms() / 2) return launch_bn<64>(a, terms, s);
  return launch_bn<128>(a, terms, s);
}

cudaError_t gemm_split_weights(const float* B, GemmLayout layout, int N, int K, void* planes_v, int64_t plane_stride,
                               cudaStream_t s, bool bf16) {
  const int64_t plane = plane_stride > 0 ? plane_stride : int64_t(N) * K;
  if (bf16) {
    dim3 grid((N + 31) / 32, (K + 31) / 32), block(32, 8);
    auto* planes = static_cast<uint16_t*>(planes_v);
    if (layout == GemmLayout::nt) split_weights_bf16_kernel<true><<<grid, block, 0, s>>>(B, planes, N, K, plane);
    else split_weights_bf16_kernel<false><<<grid, block, 0, s>>>(B, planes, N, K, plane);
    return cudaGetLastError();
  }
  float* planes = static_cast<float*>(planes_v);
  dim3 grid((N + 31) / 32, (K + 31) / 32), block(32, 8);
  if (layout == GemmLayout::nt) split_weights_kernel<true><<<grid, block, 0, s>>>(B, planes, N, K, plane);
  else split_weights_kernel<false><<<grid, block, 0, s>>>(B, planes, N, K, plane);
  return cudaGetLastError();
}

}  // namespace hs

// timing experiment only (profiles/gemm_timeline.py): gemm_tc_kernel CTA 0 stamps
extern "C" int hs_debug_gemm_timeline(long long* out, int reset) {
#if HS_DBG_GEMM_TL
  static const long long zeros[16] = {};
  if (reset) return cudaMemcpyToSymbol(hs::g_gemm_tl, zeros, sizeof(zeros)) == cudaSuccess ? 0 : 1;
  return cudaMemcpyFromSymbol(out, hs::g_gemm_tl, sizeof(long long) * 16) == cudaSuccess ? 0 : 1;
#else
  (void)out;
  (void)reset;
  return 1;
#endif
}
