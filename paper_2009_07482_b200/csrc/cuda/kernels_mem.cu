// HBM-bound DAG node kernels for sm_100a: transpose, scale, add, softmax,
// add+LayerNorm, concat.
//
// Design (B200): every kernel is a single pass over its operands with 16-byte
// vector accesses where the layout allows, coalesced along the contiguous
// dimension, and row reductions done in registers with warp shuffles (one
// warp per row; no shared-memory round trips). The instance index of a
// batched launch is a grid dimension, so one launch serves `batch` DAG
// instances; per-instance strides of 0 express shared operands.
//
// Numerics follow the CPU oracle (oracle/kernels.c): softmax = exp(s*x - max)
// with accurate expf, times 1/sum (one IEEE division per row); LayerNorm is two-pass
// (mean, then centred variance), eps added before 1/sqrt. transpose, concat
// and scale by a power of two are bit-exact.
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "launch.cuh"

namespace hs {

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int blocks_for(int64_t work, int per_block) {
  int64_t b = (work + per_block - 1) / per_block;
  return int(b < 1 ? 1 : (b > 65535 * 4 ? 65535 * 4 : b));
}

// ---------------------------------------------------------------- transpose
__global__ void transpose_kernel(const float* __restrict__ A, int64_t sA, float* __restrict__ B, int64_t sB, int R,
                                 int C) {
  pdl_launch_dependents();  // PDL (launch.cuh)
  pdl_wait();
  __shared__ float tile[32][33];
  const int64_t inst = blockIdx.z;
  A += inst * sA;
  B += inst * sB;
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    int r = r0 + i, c = c0 + threadIdx.x;
    if (r < R && c < C) tile[i][threadIdx.x] = A[int64_t(r) * C + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    int c = c0 + i, r = r0 + threadIdx.x;
    if (r < R && c < C) B[int64_t(c) * R + r] = tile[threadIdx.x][i];
  }
}

// Wide tile: 32 rows x 128 columns per block, 16-byte loads along C (each thread
// four float4, more bytes in flight than the 32 x 32 scalar tile), coalesced
// 128-byte scalar stores along R. Needs C % 4 == 0 and 16-byte aligned rows.
__global__ void transpose_wide_kernel(const float* __restrict__ A, int64_t sA, float* __restrict__ B, int64_t sB,
                                      int R, int C) {
  pdl_launch_dependents();  // PDL (launch.cuh)
  pdl_wait();
  __shared__ float tile[32][129];
  const int64_t inst = blockIdx.z;
  A += inst * sA;
  B += inst * sB;
  const int c0 = blockIdx.x * 128, r0 = blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = r0 + ty + 8 * i, c = c0 + 4 * tx;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (r < R && c < C) v = __ldg(reinterpret_cast<const float4*>(A + int64_t(r) * C + c));
    tile[ty + 8 * i][4 * tx] = v.x;
    tile[ty + 8 * i][4 * tx + 1] = v.y;
    tile[ty + 8 * i][4 * tx + 2] = v.z;
    tile[ty + 8 * i][4 * tx + 3] = v.w;
  }
  __syncthreads();
#pragma unroll 4
  for (int i = 0; i < 16; ++i) {
    const int c = c0 + ty + 8 * i, r = r0 + tx;
    if (r < R && c < C) B[int64_t(c) * R + r] = tile[tx][ty + 8 * i];
  }
}

// ---------------------------------------------------------------- elementwise
template <bool kVec>
__global__ void scale_kernel(const float* __restrict__ A, int64_t sA, float* __restrict__ B, int64_t sB, int64_t n,
                             float f) {
  pdl_launch_dependents();  // PDL (launch.cuh)
  pdl_wait();
  const int64_t inst = blockIdx.y;
  A += inst * sA;
  B += inst * sB;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  if (kVec) {
    const int64_t n4 = n >> 2;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
      float4 v = __ldg(reinterpret_cast<const float4*>(A) + i);
      v.x *= f; v.y *= f; v.z *= f; v.w *= f;
      reinterpret_cast<float4*>(B)[i] = v;
    }
  } else {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) B[i] = A[i] * f;
  }
}

template <bool kVec>
__global__ void add_kernel(const float* __restrict__ A, int64_t sA, const float* __restrict__ Bm, int64_t sB,
                           float* __restrict__ C, int64_t sC, int64_t n) {
  pdl_launch_dependents();  // PDL (launch.cuh)
  pdl_wait();
  const int64_t inst = blockIdx.y;
  A += inst * sA;
  Bm += inst * sB;
  C += inst * sC;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  if (kVec) {
    const int64_t n4 = n >> 2;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
      float4 a = __ldg(reinterpret_cast<const float4*>(A) + i);
      float4 b = __ldg(reinterpret_cast<const float4*>(Bm) + i);
      reinterpret_cast<float4*>(C)[i] = make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
    }
  } else {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) C[i] = A[i] + Bm[i];
  }
}

// ---------------------------------------------------------------- softmax
// One warp per row. kV > 0: cols == 128*kV, each lane holds kV float4 in
// registers. kV == 0: generic cols (<= 1024), scalar loads.
// One warp per row; the instance is blockIdx.y (no 64-bit division per row).
// kV > 0: cols == 128*kV, each lane holds kV float4 in registers. kV == 0:
// generic cols (<= 1024), scalar loads.
template <int kV>
__global__ void softmax_kernel(const float* __restrict__ A, int64_t sA, float* __restrict__ B, int64_t sB, int rows,
                               int cols, float f) {
  pdl_launch_dependents();  // PDL (launch.cuh)
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= rows) return;
  const int64_t inst = blockIdx.y;
  const float* a = A + inst * sA + int64_t(r) * cols;
  float* b = B + inst * sB + int64_t(r) * cols;
  if constexpr (kV > 0) {
    float4 v[kV];
    float m = -INFINITY;
#pragma unroll
    for (int j = 0; j < kV; ++j) {
      v[j] = __ldg(reinterpret_cast<const float4*>(a) + lane + 32 * j);
      v[j].x *= f; v[j].y *= f; v[j].z *= f; v[j].w *= f;
      m = fmaxf(m, fmaxf(fmaxf(v[j].x, v[j].y), fmaxf(v[j].z, v[j].w)));
    }
    m = warp_max(m);
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < kV; ++j) {
      v[j].x = expf(v[j].x - m); v[j].y = expf(v[j].y - m);
      v[j].z = expf(v[j].z - m); v[j].w = expf(v[j].w - m);
      s += (v[j].x + v[j].y) + (v[j].z + v[j].w);
    }
    const float inv = 1.f / warp_sum(s);  // one division per row, then multiplies
#pragma unroll
    for (int j = 0; j < kV; ++j) {
      v[j].x *= inv; v[j].y *= inv; v[j].z *= inv; v[j].w *= inv;
      reinterpret_cast<float4*>(b)[lane + 32 * j] = v[j];
    }
  } else {
    constexpr int kMax = 32;
    float v[kMax];
    float m = -INFINITY;
#pragma unroll
    for (int j = 0; j < kMax; ++j) {
      int c = lane + 32 * j;
      v[j] = c < cols ? a[c] * f : -INFINITY;
      m = fmaxf(m, v[j]);
    }
    m = warp_max(m);
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < kMax; ++j) {
      int c = lane + 32 * j;
      v[j] = c < cols ? expf(v[j] - m) : 0.f;
      s += v[j];
    }
    s = warp_sum(s);
#pragma unroll
    for (int j = 0; j < kMax; ++j) {
      int c = lane + 32 * j;
      if (c < cols) b[c] = v[j] / s;
    }
  }
}

// ---------------------------------------------------------------- add + LayerNorm
template <int kV>
__global__ void add_ln_kernel(const float* __restrict__ A, int64_t sA, const float* __restrict__ Bm, int64_t sB,
                              const float* __restrict__ G, int64_t sG, const float* __restrict__ Be, int64_t sBe,
                              float* __restrict__ Y, int64_t sY, int rows, int cols, float eps, int64_t total_rows) {
  pdl_launch_dependents();  // PDL (launch.cuh)
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t row = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= total_rows) return;
  const int64_t inst = row / rows, r = row % rows;
  const float* a = A + inst * sA + r * cols;
  const float* b = Bm + inst * sB + r * cols;
  const float* g = G + inst * sG;
  const float* be = Be + inst * sBe;
  float* y = Y + inst * sY + r * cols;
  const float inv_n = 1.0f / float(cols);
  if constexpr (kV > 0) {
    float4 v[kV];
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < kV; ++j) {
      float4 x = __ldg(reinterpret_cast<const float4*>(a) + lane + 32 * j);
      float4 z = __ldg(reinterpret_cast<const float4*>(b) + lane + 32 * j);
      v[j] = make_float4(x.x + z.x, x.y + z.y, x.z + z.z, x.w + z.w);
      s += (v[j].x + v[j].y) + (v[j].z + v[j].w);
    }
    const float mean = warp_sum(s) / float(cols);
    float q = 0.f;
#pragma unroll
    for (int j = 0; j < kV; ++j) {
      v[j].x -= mean; v[j].y -= mean; v[j].z -= mean; v[j].w -= mean;
      q += (v[j].x * v[j].x + v[j].y * v[j].y) + (v[j].z * v[j].z + v[j].w * v[j].w);
    }
    const float var = warp_sum(q) / float(cols);
    const float rstd = 1.0f / sqrtf(var + eps);
#pragma unroll
    for (int j = 0; j < kV; ++j) {
      float4 gg = __ldg(reinterpret_cast<const float4*>(g) + lane + 32 * j);
      float4 bb = __ldg(reinterpret_cast<const float4*>(be) + lane + 32 * j);
      float4 o = make_float4(v[j].x * rstd * gg.x + bb.x, v[j].y * rstd * gg.y + bb.y, v[j].z * rstd * gg.z + bb.z,
                             v[j].w * rstd * gg.w + bb.w);
      reinterpret_cast<float4*>(y)[lane + 32 * j] = o;
    }
  } else {
    constexpr int kMax = 32;
    float v[kMax];
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < kMax; ++j) {
      int c = lane + 32 * j;
      v[j] = c < cols ? a[c] + b[c] : 0.f;
      s += v[j];
    }
    const float mean = warp_sum(s) / float(cols);
    float q = 0.f;
#pragma unroll
    for (int j = 0; j < kMax; ++j) {
      int c = lane + 32 * j;
      v[j] = c < cols ? v[j] - mean : 0.f;
      q += v[j] * v[j];
    }
    const float var = warp_sum(q) / float(cols);
    const float rstd = 1.0f / sqrtf(var + eps);
#pragma unroll
    for (int j = 0; j < kMax; ++j) {
      int c = lane + 32 * j;
      if (c < cols) y[c] = v[j] * rstd * g[c] + be[c];
    }
    (void)inv_n;
  }
}

// ---------------------------------------------------------------- concat
struct ConcatSrc {
  const float* p[16];
  int64_t s[16];
};

template <bool kVec>
__global__ void concat_kernel(ConcatSrc src, float* __restrict__ Y, int64_t sY, int rows, int cols_each, int count) {
  pdl_launch_dependents();  // PDL (launch.cuh)
  pdl_wait();
  const int64_t inst = blockIdx.z;
  const int i = blockIdx.y;
  const float* z = src.p[i] + inst * src.s[i];
  float* y = Y + inst * sY + int64_t(i) * cols_each;
  const int64_t row_len = int64_t(cols_each) * count;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  if (kVec) {  // 32-bit index math (rows * cols_each < 2^31 per member, checked by the launcher)
    const int c4 = cols_each >> 2;
    const int n4 = rows * c4;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n4; t += int(stride)) {
      const int r = t / c4, c = t - r * c4;
      float4 v = __ldg(reinterpret_cast<const float4*>(z + int64_t(r) * cols_each) + c);
      *reinterpret_cast<float4*>(y + int64_t(r) * row_len + c * 4) = v;
    }
  } else {
    const int64_t n = int64_t(rows) * cols_each;
    for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < n; t += stride) {
      int64_t r = t / cols_each, c = t % cols_each;
      y[r * row_len + c] = z[r * cols_each + c];
    }
  }
}

}  // namespace

cudaError_t transpose(const float* A, int64_t sA, float* B, int64_t sB, int R, int C, int batch, cudaStream_t s) {
  if (C % 4 == 0 && sA % 4 == 0 && aligned16(A)) {
    dim3 grid((C + 127) / 128, (R + 31) / 32, batch), block(32, 8);
    HS_TRY(launch_node(transpose_wide_kernel, dim3(grid), dim3(block), 0, s, 1, A, sA, B, sB, R, C));
  } else {
    dim3 grid((C + 31) / 32, (R + 31) / 32, batch), block(32, 8);
    HS_TRY(launch_node(transpose_kernel, dim3(grid), dim3(block), 0, s, 1, A, sA, B, sB, R, C));
  }
  return cudaGetLastError();
}

cudaError_t scale(const float* A, int64_t sA, float* B, int64_t sB, int64_t n, float f, int batch, cudaStream_t s) {
  bool vec = n % 4 == 0 && sA % 4 == 0 && sB % 4 == 0 && aligned16(A) && aligned16(B);
  dim3 grid(blocks_for(vec ? n / 4 : n, kThreads), batch);
  if (vec) HS_TRY(launch_node(scale_kernel<true>, dim3(grid), dim3(kThreads), 0, s, 1, A, sA, B, sB, n, f));
  else HS_TRY(launch_node(scale_kernel<false>, dim3(grid), dim3(kThreads), 0, s, 1, A, sA, B, sB, n, f));
  return cudaGetLastError();
}

cudaError_t add(const float* A, int64_t sA, const float* B, int64_t sB, float* C, int64_t sC, int64_t n, int batch,
                cudaStream_t s) {
  bool vec = n % 4 == 0 && sA % 4 == 0 && sB % 4 == 0 && sC % 4 == 0 && aligned16(A) && aligned16(B) && aligned16(C);
  dim3 grid(blocks_for(vec ? n / 4 : n, kThreads), batch);
  if (vec) HS_TRY(launch_node(add_kernel<true>, dim3(grid), dim3(kThreads), 0, s, 1, A, sA, B, sB, C, sC, n));
  else HS_TRY(launch_node(add_kernel<false>, dim3(grid), dim3(kThreads), 0, s, 1, A, sA, B, sB, C, sC, n));
  return cudaGetLastError();
}

cudaError_t softmax(const float* A, int64_t sA, float* B, int64_t sB, int rows, int cols, float f, int batch,
                    cudaStream_t s) {
  if (cols > 1024 || cols < 1 || batch > 65535) return cudaErrorInvalidValue;
  const int rows_per_block = kThreads / 32;
  dim3 grid(unsigned((rows + rows_per_block - 1) / rows_per_block), unsigned(batch));
  bool vec = cols % 128 == 0 && sA % 4 == 0 && sB % 4 == 0 && aligned16(A) && aligned16(B);
  int v = vec ? cols / 128 : 0;
  switch (v) {
    case 1: HS_TRY(launch_node(softmax_kernel<1>, dim3(grid), dim3(kThreads), 0, s, 1, A, sA, B, sB, rows, cols, f)); break;
    case 2: HS_TRY(launch_node(softmax_kernel<2>, dim3(grid), dim3(kThreads), 0, s, 1, A, sA, B, sB, rows, cols, f)); break;
    case 4: HS_TRY(launch_node(softmax_kernel<4>, dim3(grid), dim3(kThreads), 0, s, 1, A, sA, B, sB, rows, cols, f)); break;
    case 8: HS_TRY(launch_node(softmax_kernel<8>, dim3(grid), dim3(kThreads), 0, s, 1, A, sA, B, sB, rows, cols, f)); break;
    default: HS_TRY(launch_node(softmax_kernel<0>, dim3(grid), dim3(kThreads), 0, s, 1, A, sA, B, sB, rows, cols, f)); break;
  }
  return cudaGetLastError();
}

cudaError_t add_layernorm(const float* A, int64_t sA, const float* B, int64_t sB, const float* gamma, int64_t sG,
                          const float* beta, int64_t sBt, float* Y, int64_t sY, int rows, int cols, float eps,
                          int batch, cudaStream_t s) {
  if (cols > 1024 || cols < 1) return cudaErrorInvalidValue;
  const int64_t total = int64_t(rows) * batch;
  const int rows_per_block = kThreads / 32;
  dim3 grid(unsigned((total + rows_per_block - 1) / rows_per_block));
  bool vec = cols % 128 == 0 && sA % 4 == 0 && sB % 4 == 0 && sG % 4 == 0 && sBt % 4 == 0 && sY % 4 == 0 &&
             aligned16(A) && aligned16(B) && aligned16(gamma) && aligned16(beta) && aligned16(Y);
  int v = vec ? cols / 128 : 0;
  switch (v) {
    case 1: HS_TRY(launch_node(add_ln_kernel<1>, dim3(grid), dim3(kThreads), 0, s, 1, A, sA, B, sB, gamma, sG, beta, sBt, Y, sY, rows, cols, eps, total)); break;
    case 2: HS_TRY(launch_node(add_ln_kernel<2>, dim3(grid), dim3(kThreads), 0, s, 1, A, sA, B, sB, gamma, sG, beta, sBt, Y, sY, rows, cols, eps, total)); break;
    case 4: HS_TRY(launch_node(add_ln_kernel<4>, dim3(grid), dim3(kThreads), 0, s, 1, A, sA, B, sB, gamma, sG, beta, sBt, Y, sY, rows, cols, eps, total)); break;
    case 8: HS_TRY(launch_node(add_ln_kernel<8>, dim3(grid), dim3(kThreads), 0, s, 1, A, sA, B, sB, gamma, sG, beta, sBt, Y, sY, rows, cols, eps, total)); break;
    default: HS_TRY(launch_node(add_ln_kernel<0>, dim3(grid), dim3(kThreads), 0, s, 1, A, sA, B, sB, gamma, sG, beta, sBt, Y, sY, rows, cols, eps, total)); break;
  }
  return cudaGetLastError();
}

cudaError_t concat(const float* const* Z, const int64_t* sZ, int count, float* Y, int64_t sY, int rows, int cols_each,
                   int batch, cudaStream_t s) {
  if (count < 1 || count > 16) return cudaErrorInvalidValue;
  ConcatSrc src{};
  bool vec = cols_each % 4 == 0 && sY % 4 == 0 && aligned16(Y);
  for (int i = 0; i < count; ++i) {
    src.p[i] = Z[i];
    src.s[i] = sZ[i];
    vec = vec && sZ[i] % 4 == 0 && aligned16(Z[i]);
  }
  vec = vec && int64_t(rows) * cols_each < (int64_t(1) << 31);
  const int64_t work = vec ? int64_t(rows) * (cols_each / 4) : int64_t(rows) * cols_each;
  dim3 grid(blocks_for(work, kThreads), count, batch);
  if (vec) HS_TRY(launch_node(concat_kernel<true>, dim3(grid), dim3(kThreads), 0, s, 1, src, Y, sY, rows, cols_each, count));
  else HS_TRY(launch_node(concat_kernel<false>, dim3(grid), dim3(kThreads), 0, s, 1, src, Y, sY, rows, cols_each, count));
  return cudaGetLastError();
}

}  // namespace hs
