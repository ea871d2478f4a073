// Launchers for the DAG node kernels (sm_100a). All pointers are device
// pointers; every buffer carries a per-instance stride in elements (0 means
// the buffer is shared by all `batch` instances, e.g. resident weights).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace hs {

enum class GemmLayout { nn, nt };  // B is [K,N] row-major (nn) or [N,K] row-major (nt)

struct GemmArgs {
  const float* A;
  int64_t sA;
  const float* B;
  int64_t sB;
  float* C;
  int64_t sC;
  int M, N, K;
  int batch;
  GemmLayout layout;
  bool relu;
  // Optional: resident B pre-split into K-major tf32 planes [2][N][K] (hi, lo)
  // by gemm_split_weights; then B is fed to the tensor cores by TMA directly.
  const float* Bplanes = nullptr;
  // Grouped launch of n_out sibling GEMMs sharing A: N is the total column
  // count, Bplanes their concatenated planes, member m writes Cs[m] (stride sCs[m]).
  int n_out = 0;
  float* Cs[4] = {nullptr, nullptr, nullptr, nullptr};
  int64_t sCs[4] = {0, 0, 0, 0};
  // Bplanes hold bf16 hi/lo (math BF16x3) instead of tf32 hi/lo.
  int bf16 = 0;
  // Row stride of C in elements (0 = N, or the member width for grouped launches).
  int64_t ldc = 0;
  // 1 = row softmax of (A·B)·escale over the N columns (N <= 128, one tile row).
  int softmax = 0;
  float escale = 1.f;
  // no split-K (HS_FLAG_DETERMINISTIC): bit-reproducible single-instance launches
  bool deterministic = false;
};

// planes: hi at planes[n*K + k], lo at planes[plane_stride + n*K + k]
cudaError_t gemm_split_weights(const float* B, GemmLayout layout, int N, int K, void* planes, int64_t plane_stride,
                               cudaStream_t s, bool bf16 = false);

// math: 0 = TF32x3 (tcgen05), 1 = TF32 (tcgen05), 2 = fp32 SIMT
cudaError_t gemm_tcgen05(const GemmArgs& a, int terms, cudaStream_t s);
cudaError_t gemm_simt(const GemmArgs& a, cudaStream_t s);
// true when the tcgen05 path supports this shape/alignment
bool gemm_tcgen05_supported(const GemmArgs& a);

// Fused attention head (HS_OP_ATTN_HEAD): Z = softmax_row(scale · Q Kᵀ) · V · W per
// instance; Q, K, V are [S, dk] (S <= 128, dk = 64), W is [dk, dw] (dw = 64)
// pre-split into tf32 hi/lo planes [2][dw][dk] (gemm_split_weights format 0).
// Z rows are ldz elements apart (0 = dw) so Z can be a column block of a concat.
struct AttnArgs {
  const float* Q;
  int64_t sQ;
  const float* K;
  int64_t sK;
  const float* V;
  int64_t sV;
  const void* Wplanes;
  float* Z;
  int64_t sZ;
  int64_t ldz;
  int S, dk, dw, batch;
  float scale;
};
bool attn_head_supported(const AttnArgs& a);
cudaError_t attn_head(const AttnArgs& a, int terms, cudaStream_t s);

// Whole transformer head (HS_OP_HEAD): [Q|K|V] = X · Wqkv, Z = softmax_row(scale · Q Kᵀ)
// · V · Wh per instance. X is [S, D] (S <= 128, D % 32 == 0); Wqkv is pre-split into
// tf32 hi/lo planes [2][3 dk][D] (q | k | v rows, gemm_split_weights format 0, plane
// stride 3 dk D); Wh planes [2][dk][dk]; dk = 64. Z rows are ldz apart (0 = dk).
struct HeadArgs {
  const float* X;
  int64_t sX;
  const void* Wqkv;
  const void* Wh;
  float* Z;
  int64_t sZ;
  int64_t ldz;
  int S, D, dk, batch;
  float scale;
};
bool head_fused_supported(const HeadArgs& a);
cudaError_t head_fused(const HeadArgs& a, int terms, cudaStream_t s);

cudaError_t transpose(const float* A, int64_t sA, float* B, int64_t sB, int R, int C, int batch, cudaStream_t s);
cudaError_t scale(const float* A, int64_t sA, float* B, int64_t sB, int64_t n, float f, int batch, cudaStream_t s);
cudaError_t add(const float* A, int64_t sA, const float* B, int64_t sB, float* C, int64_t sC, int64_t n, int batch,
                cudaStream_t s);
cudaError_t softmax(const float* A, int64_t sA, float* B, int64_t sB, int rows, int cols, float f, int batch,
                    cudaStream_t s);
cudaError_t add_layernorm(const float* A, int64_t sA, const float* B, int64_t sB, const float* gamma, int64_t sG,
                          const float* beta, int64_t sBt, float* Y, int64_t sY, int rows, int cols, float eps,
                          int batch, cudaStream_t s);
cudaError_t concat(const float* const* Z, const int64_t* sZ, int count, float* Y, int64_t sY, int rows, int cols_each,
                   int batch, cudaStream_t s);

}  // namespace hs
