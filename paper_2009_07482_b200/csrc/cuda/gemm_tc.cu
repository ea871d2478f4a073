// tcgen05 / TMEM / TMA GEMM for sm_100a with an fp32-accurate 3xTF32 mode.
//
//   C[M,N] (+ReLU) = A[M,K] · B        B = [K,N] row-major (nn) or [N,K] (nt)
//
// Per CTA: one 128 x BN output tile, accumulator in TMEM (BN fp32 columns).
// Warp roles (256 threads):
//   warp 0      TMA producer: fp32 A/B tiles (K-block of 32) -> staging ring
//   warp 1      MMA issuer: one elected lane issues tcgen05.mma.kind::tf32
//   warp 2      TMEM allocator
//   warps 4..7  converters during the main loop: staging fp32 -> canonical
//               K-major SWIZZLE_128B operand planes, split x = hi + lo with
//               hi = cvt.rna.tf32(x), lo = x - hi (exact); then the epilogue
//               (tcgen05.ld 32x32b -> registers -> ReLU -> global).
// 3xTF32: D += Ahi·Bhi + Ahi·Blo + Alo·Bhi (the Alo·Blo term, ~2^-22
// relative, is dropped). TF32 mode (terms=1) issues only Ahi·Bhi.
//
// Pipelines (mbarriers): staging full/empty (TMA <-> converters), operand
// full/empty (converters <-> MMA, released by tcgen05.commit), accumulator
// full (MMA -> epilogue). TMA zero-fills out-of-bounds boxes, so ragged M, N
// and K tails need no special casing in the main loop.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <mutex>

#include "kernels.cuh"

namespace hs {

namespace {

constexpr int BM = 128;
constexpr int BK = 32;  // fp32 elements per K-block = one 128-byte swizzle row
constexpr int kStages = 2;
constexpr int kThreads = 256;

// ----------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::
          "r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// Shared-memory matrix descriptor: K-major, SWIZZLE_128B, 8-row core groups
// 1024 bytes apart (SBO), version 1 (sm_100).
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
  return uint64_t((addr >> 4) & 0x3FFFu) | (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) | (uint64_t(1) << 46) |
         (uint64_t(2) << 61);
}
// Instruction descriptor: D=f32, A=B=tf32, both K-major, M=128, N=n.
__host__ __device__ constexpr uint32_t instr_desc_tf32(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(BM >> 4) << 24);
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
__device__ __forceinline__ float4 lds128(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ float lds32(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t addr, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
// Byte offset of 16-byte chunk `kc` (0..7) of row `r` in a K-major SW128 tile.
__device__ __forceinline__ uint32_t sw128(int r, int kc) {
  return uint32_t((r >> 3) * 1024 + (r & 7) * 128 + ((kc ^ (r & 7)) << 4));
}

template <int kTerms>
__device__ __forceinline__ void split_store(uint32_t hi_base, uint32_t lo_base, uint32_t off, float4 x) {
  float4 h = make_float4(tf32_rna(x.x), tf32_rna(x.y), tf32_rna(x.z), tf32_rna(x.w));
  sts128(hi_base + off, h);
  if constexpr (kTerms > 1) sts128(lo_base + off, make_float4(x.x - h.x, x.y - h.y, x.z - h.z, x.w - h.w));
}

template <int BN>
struct Smem {
  static constexpr int kStageA = BM * BK * 4;        // fp32 staging, row-major [128][32]
  static constexpr int kStageB = BN * BK * 4;        // [BN][32] (nt) or [32][BN] (nn)
  static constexpr int kPlaneA = BM * 128;           // one SW128 plane: 128 rows x 128 B
  static constexpr int kPlaneB = BN * 128;
  static constexpr int kStaging = kStageA + kStageB;
  static constexpr int kOperand = 2 * kPlaneA + 2 * kPlaneB;  // hi + lo for A and B
  static constexpr int kBarriers = 1024;
  static constexpr int kTotal = kStages * (kStaging + kOperand) + kBarriers + 1024;  // + alignment slack
};

template <int BN, bool kNT, int kTerms>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, float* C,
                   int64_t sC, int M, int N, int K, int a_batched, int b_batched, int relu) {
  using L = Smem<BN>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t staging = base;
  const uint32_t operand = staging + kStages * L::kStaging;
  const uint32_t bars = operand + kStages * L::kOperand;
  // barrier layout (8 bytes each)
  auto st_full = [&](int s) { return bars + 8u * uint32_t(s); };
  auto st_empty = [&](int s) { return bars + 8u * uint32_t(kStages + s); };
  auto op_full = [&](int s) { return bars + 8u * uint32_t(2 * kStages + s); };
  auto op_empty = [&](int s) { return bars + 8u * uint32_t(3 * kStages + s); };
  const uint32_t acc_full = bars + 8u * uint32_t(4 * kStages);
  const uint32_t tmem_slot = bars + 8u * uint32_t(4 * kStages + 1);
  uint32_t* tmem_slot_ptr = reinterpret_cast<uint32_t*>(smem_raw + (tmem_slot - smem_u32(smem_raw)));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * BN, m0 = blockIdx.y * BM, inst = blockIdx.z;
  const int nk = (K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(st_full(s), 1);
      mbar_init(st_empty(s), 4);
      mbar_init(op_full(s), 4);
      mbar_init(op_empty(s), 1);
    }
    mbar_init(acc_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tmem_slot), "r"(BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot_ptr;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      const int ia = a_batched ? inst : 0, ib = b_batched ? inst : 0;
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % kStages;
        const uint32_t ph = uint32_t(kb / kStages) & 1u;
        mbar_wait(st_empty(s), ph ^ 1u);
        const uint32_t sa = staging + uint32_t(s) * L::kStaging, sb = sa + L::kStageA;
        mbar_expect_tx(st_full(s), L::kStaging);
        tma_load_3d(sa, &tmA, st_full(s), kb * BK, m0, ia);
        if (kNT) tma_load_3d(sb, &tmB, st_full(s), kb * BK, n0, ib);
        else tma_load_3d(sb, &tmB, st_full(s), n0, kb * BK, ib);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = instr_desc_tf32(BN);
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % kStages;
        const uint32_t ph = uint32_t(kb / kStages) & 1u;
        mbar_wait(op_full(s), ph);
        tc_fence_after();
        const uint32_t a_hi = operand + uint32_t(s) * L::kOperand;
        const uint32_t a_lo = a_hi + L::kPlaneA;
        const uint32_t b_hi = a_lo + L::kPlaneA;
        const uint32_t b_lo = b_hi + L::kPlaneB;
#pragma unroll
        for (int kk = 0; kk < BK / 8; ++kk) {  // K = 8 tf32 per instruction = 32 bytes
          const uint32_t koff = uint32_t(kk) * 32u;
          const uint32_t acc = (kb | kk) ? 1u : 0u;
          if constexpr (kTerms > 1) {
            mma_tf32(tmem, smem_desc(a_lo + koff), smem_desc(b_hi + koff), idesc, acc);
            mma_tf32(tmem, smem_desc(a_hi + koff), smem_desc(b_lo + koff), idesc, 1u);
            mma_tf32(tmem, smem_desc(a_hi + koff), smem_desc(b_hi + koff), idesc, 1u);
          } else {
            mma_tf32(tmem, smem_desc(a_hi + koff), smem_desc(b_hi + koff), idesc, acc);
          }
        }
        mma_commit(op_empty(s));  // operand slot free once these MMAs have read it
      }
      mma_commit(acc_full);
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ converters
    const int t = threadIdx.x - 128;  // 0..127
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % kStages;
      const uint32_t ph = uint32_t(kb / kStages) & 1u;
      mbar_wait(st_full(s), ph);
      mbar_wait(op_empty(s), ph ^ 1u);
      const uint32_t sa = staging + uint32_t(s) * L::kStaging, sb = sa + L::kStageA;
      const uint32_t a_hi = operand + uint32_t(s) * L::kOperand;
      const uint32_t a_lo = a_hi + L::kPlaneA;
      const uint32_t b_hi = a_lo + L::kPlaneA;
      const uint32_t b_lo = b_hi + L::kPlaneB;
      // A: staging row-major [128][32] -> SW128 planes. 8 threads per 128-byte row.
#pragma unroll
      for (int j = 0; j < (BM * 8) / 128; ++j) {
        const int id = t + 128 * j, r = id >> 3, kc = id & 7;
        split_store<kTerms>(a_hi, a_lo, sw128(r, kc), lds128(sa + uint32_t(r * 128 + kc * 16)));
      }
      if constexpr (kNT) {
#pragma unroll
        for (int j = 0; j < (BN * 8) / 128; ++j) {
          const int id = t + 128 * j, r = id >> 3, kc = id & 7;
          split_store<kTerms>(b_hi, b_lo, sw128(r, kc), lds128(sb + uint32_t(r * 128 + kc * 16)));
        }
      } else {
        // staging [32 k][BN n]: gather 4 consecutive k of one column n (conflict-free:
        // consecutive threads take consecutive n), write one 16-byte K-major chunk.
#pragma unroll
        for (int j = 0; j < (BN * 8) / 128; ++j) {
          const int id = t + 128 * j, n = id % BN, kc = id / BN;
          const uint32_t src = sb + uint32_t((kc * 4) * BN + n) * 4u;
          float4 x = make_float4(lds32(src), lds32(src + BN * 4), lds32(src + 2 * BN * 4), lds32(src + 3 * BN * 4));
          split_store<kTerms>(b_hi, b_lo, sw128(n, kc), x);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> async (MMA) reads
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(st_empty(s));
        mbar_arrive(op_full(s));
      }
    }
    // ------------------------------------------------------------ epilogue
    mbar_wait(acc_full, 0);
    tc_fence_after();
    const int q = warp - 4;  // TMEM lane quarter accessible to this warp
    const int row = m0 + q * 32 + lane;
    float* crow = C + int64_t(inst) * sC + int64_t(row) * N;
#pragma unroll 1
    for (int cb = 0; cb < BN / 32; ++cb) {
      uint32_t r[32];
      const uint32_t taddr = tmem + (uint32_t(q * 32) << 16) + uint32_t(cb * 32);
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
            "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
            "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      const int c0 = n0 + cb * 32;
      if (row < M) {
        if (c0 + 32 <= N && (N & 3) == 0) {
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            float4 v = make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]), __uint_as_float(r[j + 2]),
                                   __uint_as_float(r[j + 3]));
            if (relu) {
              v.x = fmaxf(v.x, 0.f); v.y = fmaxf(v.y, 0.f); v.z = fmaxf(v.z, 0.f); v.w = fmaxf(v.w, 0.f);
            }
            *reinterpret_cast<float4*>(crow + c0 + j) = v;
          }
        } else {
          for (int j = 0; j < 32; ++j) {
            if (c0 + j >= N) break;
            float v = __uint_as_float(r[j]);
            crow[c0 + j] = relu ? fmaxf(v, 0.f) : v;
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(BN));
  }
}

// ----------------------------------------------------------------- host side
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return EncodeTiledFn(nullptr);
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// 3-D fp32 tensor map: dims {d0 (contiguous), d1, d2}, byte strides {s1, s2}.
bool make_map(CUtensorMap* m, const float* ptr, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1, uint64_t s2,
              uint32_t b0, uint32_t b1) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {s1, s2};
  cuuint32_t box[3] = {b0, b1, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(ptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int BN, bool kNT, int kTerms>
cudaError_t launch(const GemmArgs& a, cudaStream_t s) {
  auto kernel = gemm_tc_kernel<BN, kNT, kTerms>;
  constexpr int smem = Smem<BN>::kTotal;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [&] { attr_err = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); });
  if (attr_err != cudaSuccess) return attr_err;
  const uint64_t nA = a.sA ? uint64_t(a.batch) : 1, nB = a.sB ? uint64_t(a.batch) : 1;
  const uint64_t sA = (a.sA ? uint64_t(a.sA) : uint64_t(a.M) * a.K) * 4;
  CUtensorMap mA, mB;
  if (!make_map(&mA, a.A, uint64_t(a.K), uint64_t(a.M), nA, uint64_t(a.K) * 4, sA, BK, BM)) return cudaErrorInvalidValue;
  bool ok;
  if (kNT) {
    const uint64_t sB = (a.sB ? uint64_t(a.sB) : uint64_t(a.N) * a.K) * 4;
    ok = make_map(&mB, a.B, uint64_t(a.K), uint64_t(a.N), nB, uint64_t(a.K) * 4, sB, BK, BN);
  } else {
    const uint64_t sB = (a.sB ? uint64_t(a.sB) : uint64_t(a.N) * a.K) * 4;
    ok = make_map(&mB, a.B, uint64_t(a.N), uint64_t(a.K), nB, uint64_t(a.N) * 4, sB, BN, BK);
  }
  if (!ok) return cudaErrorInvalidValue;
  dim3 grid((a.N + BN - 1) / BN, (a.M + BM - 1) / BM, a.batch);
  kernel<<<grid, kThreads, smem, s>>>(mA, mB, a.C, a.sC, a.M, a.N, a.K, a.sA != 0, a.sB != 0, a.relu ? 1 : 0);
  return cudaGetLastError();
}

template <int BN>
cudaError_t launch_bn(const GemmArgs& a, int terms, cudaStream_t s) {
  const bool nt = a.layout == GemmLayout::nt;
  if (terms > 1) return nt ? launch<BN, true, 3>(a, s) : launch<BN, false, 3>(a, s);
  return nt ? launch<BN, true, 1>(a, s) : launch<BN, false, 1>(a, s);
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace

bool gemm_tcgen05_supported(const GemmArgs& a) {
  if (a.M < 1 || a.N < 1 || a.K < 1 || a.batch < 1) return false;
  if (a.K % 4 || (a.layout == GemmLayout::nn && a.N % 4)) return false;
  if (a.sA % 4 || a.sB % 4 || a.sC % 4) return false;
  if (!aligned16(a.A) || !aligned16(a.B) || !aligned16(a.C)) return false;
  if (a.batch > 65535) return false;
  return encode_fn() != nullptr;
}

cudaError_t gemm_tcgen05(const GemmArgs& a, int terms, cudaStream_t s) {
  if (a.N <= 64) return launch_bn<64>(a, terms, s);
  return launch_bn<128>(a, terms, s);
}

}  // namespace hs
