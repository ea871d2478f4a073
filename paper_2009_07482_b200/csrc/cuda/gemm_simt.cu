// CUDA-core fp32 GEMM (HS_MATH_FP32_SIMT). Diagnostic path: an on-device
// fp32 reference for the tcgen05 kernels and a fallback for shapes the
// tensor-core path rejects (K or N not a multiple of 4). Same contract as
// the tcgen05 kernel: C = A·B (B row-major [K,N] or [N,K]), optional ReLU,
// batched over instances with per-operand strides and an optional output row
// stride (ldc). The softmax epilogue is tcgen05-only.
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "launch.cuh"

namespace hs {

namespace {

constexpr int BM = 64, BN = 64, BK = 16;

template <bool kNT>
__global__ void __launch_bounds__(256) gemm_simt_kernel(GemmArgs p) {
  pdl_launch_dependents();  // PDL (launch.cuh)
  pdl_wait();
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int64_t inst = blockIdx.z;
  const float* A = p.A + inst * p.sA;
  const float* B = p.B + inst * p.sB;
  float* C = p.C + inst * p.sC;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < p.K; k0 += BK) {
    for (int i = threadIdx.x; i < BM * BK; i += 256) {
      int r = i / BK, k = i % BK;
      int gm = m0 + r, gk = k0 + k;
      As[k][r] = (gm < p.M && gk < p.K) ? A[int64_t(gm) * p.K + gk] : 0.f;
    }
    for (int i = threadIdx.x; i < BN * BK; i += 256) {
      int k, c;
      if (kNT) { c = i / BK; k = i % BK; } else { k = i / BN; c = i % BN; }
      int gn = n0 + c, gk = k0 + k;
      float v = 0.f;
      if (gn < p.N && gk < p.K) v = kNT ? B[int64_t(gn) * p.K + gk] : B[int64_t(gk) * p.N + gn];
      Bs[k][c] = v;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[k][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[k][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int gm = m0 + ty * 4 + i;
    if (gm >= p.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int gn = n0 + tx * 4 + j;
      if (gn >= p.N) continue;
      float v = acc[i][j];
      if (p.relu) v = fmaxf(v, 0.f);
      C[int64_t(gm) * (p.ldc ? p.ldc : p.N) + gn] = v;
    }
  }
}

}  // namespace

cudaError_t gemm_simt(const GemmArgs& a, cudaStream_t s) {
  dim3 grid((a.N + BN - 1) / BN, (a.M + BM - 1) / BM, a.batch);
  if (a.layout == GemmLayout::nt) HS_TRY(launch_node(gemm_simt_kernel<true>, dim3(grid), dim3(256), 0, s, 1, a));
  else HS_TRY(launch_node(gemm_simt_kernel<false>, dim3(grid), dim3(256), 0, s, 1, a));
  return cudaGetLastError();
}

}  // namespace hs
