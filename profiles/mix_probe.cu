// Probe: can one kernel run cta_group::2 (CTA-pair) and cta_group::1 tcgen05 MMAs
// side by side? A cluster of 2 allocates 512 TMEM columns with cta_group::2; the
// leader issues pair MMAs (M = 256: 128 rows per CTA, N = 64, B rows split 32/32)
// into columns [0, 64) while each CTA issues its own cta_group::1 MMAs (M = 128,
// N = 64) into columns [128, 192), interleaved over many iterations. Inputs are
// small integers (exact in tf32), so both results are checked exactly.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 [-DMIX_SPLIT=1] -o /tmp/mix_probe profiles/mix_probe.cu -lcuda
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#include "../paper_2009_07482_b200/csrc/cuda/tc_common.cuh"

using namespace hs::tc;

constexpr int kIters = 64;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    mix_probe(const float* A2, const float* B2, const float* A1, const float* B1, float* D2, float* D1) {
  __shared__ __align__(1024) uint8_t smem[2 * 8192 + 64];
  const uint32_t base = smem_u32(smem);
  const uint32_t sB2 = base, sB1 = base + 8192, bar2 = base + 16384, bar1 = bar2 + 8, slot = bar2 + 16;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, row = threadIdx.x;
  const uint32_t rank = cluster_ctarank();
  if (threadIdx.x == 0) {
    mbar_init(bar2, 1);
    mbar_init(bar1, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(slot), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  // B operands, K-major SW128 (8 k-columns = 32 bytes used per row): pair B = this CTA's
  // 32 rows of the 64, single B = all 64 rows
  for (int n = threadIdx.x; n < 64; n += blockDim.x)
    for (int c = 0; c < 2; ++c) {
      const float* src2 = B2 + (int(rank) * 32 + n) * 8 + 4 * c;
      const float* src1 = B1 + (int(rank) * 64 + n) * 8 + 4 * c;
      if (n < 32) sts128(sB2 + sw128(n, c), make_float4(src2[0], src2[1], src2[2], src2[3]));
      sts128(sB1 + sw128(n, c), make_float4(src1[0], src1[1], src1[2], src1[3]));
    }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem + 16384 + 16);
  // A operands in TMEM: pair A (this CTA's 128 rows) at [256, 264), single A at [320, 328)
  {
    const uint32_t lb = tmem + (uint32_t(warp * 32) << 16);
    uint32_t a2[16] = {}, a1[16] = {};
    for (int k = 0; k < 8; ++k) {
      a2[k] = __float_as_uint(A2[(int(rank) * 128 + row) * 8 + k]);
      a1[k] = __float_as_uint(A1[(int(rank) * 128 + row) * 8 + k]);
    }
    tmem_st16(lb + 256, a2);
    tmem_st16(lb + 320, a1);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
#ifndef MIX_SPLIT  // MIX_SPLIT=1: the single-CTA MMAs come from another warp (own issuer thread)
#define MIX_SPLIT 0
#endif
  const uint32_t id2 = instr_desc_tf32(64, 256), id1 = instr_desc_tf32(64, 128);
  if (warp == 1) {
    for (int it = 0; it < kIters; ++it) {
      if (elect_one()) {
        if (rank == 0) mma_pair_tf32_ts(tmem + 0, tmem + 256, smem_desc(sB2), id2, it ? 1u : 0u);
        if (!MIX_SPLIT) mma_tf32_ts(tmem + 128, tmem + 320, smem_desc(sB1), id1, it ? 1u : 0u);
      }
      __syncwarp();
    }
    if (elect_one()) {
      if (rank == 0) mma_commit_pair(bar2);
      if (!MIX_SPLIT) mma_commit(bar1);
    }
    __syncwarp();
  } else if (warp == 2 && MIX_SPLIT) {
    for (int it = 0; it < kIters; ++it) {
      if (elect_one()) mma_tf32_ts(tmem + 128, tmem + 320, smem_desc(sB1), id1, it ? 1u : 0u);
      __syncwarp();
    }
    if (elect_one()) mma_commit(bar1);
    __syncwarp();
  }
  mbar_wait(bar2, 0);
  mbar_wait(bar1, 0);
  tc_fence_after();
  {
    const uint32_t lb = tmem + (uint32_t(warp * 32) << 16);
    uint32_t r[32];
    for (int h = 0; h < 2; ++h) {
      tmem_ld32(lb + uint32_t(32 * h), r);
      for (int j = 0; j < 32; ++j) D2[(int(rank) * 128 + row) * 64 + 32 * h + j] = __uint_as_float(r[j]);
      tmem_ld32(lb + 128u + uint32_t(32 * h), r);
      for (int j = 0; j < 32; ++j) D1[(int(rank) * 128 + row) * 64 + 32 * h + j] = __uint_as_float(r[j]);
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

int main() {
  // pair: D2[r][n] = it * sum_k A2[r][k] B2[n][k]  (r over 256 rows = 2 CTAs x 128)
  // single: D1[cta][r][n] = it * sum_k A1[cta][r][k] B1[cta][n][k]
  std::vector<float> A2(256 * 8), B2(64 * 8), A1(256 * 8), B1(2 * 64 * 8);
  for (size_t i = 0; i < A2.size(); ++i) A2[i] = float(int(i * 7 % 5) - 2);
  for (size_t i = 0; i < B2.size(); ++i) B2[i] = float(int(i * 3 % 7) - 3);
  for (size_t i = 0; i < A1.size(); ++i) A1[i] = float(int(i * 11 % 9) - 4);
  for (size_t i = 0; i < B1.size(); ++i) B1[i] = float(int(i * 5 % 3) - 1);
  float *dA2, *dB2, *dA1, *dB1, *dD2, *dD1;
  cudaMalloc(&dA2, A2.size() * 4);
  cudaMalloc(&dB2, B2.size() * 4);
  cudaMalloc(&dA1, A1.size() * 4);
  cudaMalloc(&dB1, B1.size() * 4);
  cudaMalloc(&dD2, 256 * 64 * 4);
  cudaMalloc(&dD1, 256 * 64 * 4);
  cudaMemcpy(dA2, A2.data(), A2.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB2, B2.data(), B2.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dA1, A1.data(), A1.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB1, B1.data(), B1.size() * 4, cudaMemcpyHostToDevice);
  int bad2 = 0, bad1 = 0;
  for (int rep = 0; rep < 200; ++rep) {
    cudaMemset(dD2, 0, 256 * 64 * 4);
    cudaMemset(dD1, 0, 256 * 64 * 4);
    mix_probe<<<2 * 74, 128>>>(dA2, dB2, dA1, dB1, dD2, dD1);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("FAIL: %s\n", cudaGetErrorString(e));
      return 1;
    }
    std::vector<float> D2(256 * 64), D1(256 * 64);
    cudaMemcpy(D2.data(), dD2, D2.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(D1.data(), dD1, D1.size() * 4, cudaMemcpyDeviceToHost);
    for (int r = 0; r < 256; ++r)
      for (int n = 0; n < 64; ++n) {
        float s2 = 0, s1 = 0;
        const int cta = r / 128;
        for (int k = 0; k < 8; ++k) {
          s2 += A2[r * 8 + k] * B2[n * 8 + k];
          s1 += A1[r * 8 + k] * B1[(cta * 64 + n) * 8 + k];
        }
        bad2 += D2[r * 64 + n] != kIters * s2;
        bad1 += D1[r * 64 + n] != kIters * s1;
      }
  }
  printf("%s: pair mismatches %d, single mismatches %d (200 launches x 74 clusters, last cluster checked)\n",
         bad2 || bad1 ? "FAIL" : "PASS", bad2, bad1);
  return bad2 || bad1;
}
