/*
 * TEST INFRASTRUCTURE ONLY — the CPU checker for the DAG node kernels.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * this library (oracle/liboracle.so); the product never links it.
 *
 * Plain fp32 C restatement of the node semantics:
 *   gemm       PAPER.md:232-241 (OpenCL `gemm(A,B,C,M,N,K)`): C[i][j] accumulates
 *              A[i][k]*B[k][j] for k = 0..K-1 in fp32, sequential k. The loop is
 *              written i-k-j so it vectorises across j, but every C[i][j] still
 *              sees exactly the paper's k-ascending sequence of fp32 mul+add
 *              (compiled without FMA contraction: -std=c11 => -ffp-contract=off).
 *   gemm_nt    same with B[j][k]; gemm_relu = max(0, gemm)  (PAPER.md:323 QK^T)
 *   transpose  B[c][r] = A[r][c] (bit-exact)
 *   scale      B = A * s
 *   softmax    y = exp(s*x - max) / sum, sequential sum (PAPER.md:323 Softmax)
 *   add        C = A + B
 *   add_ln     v = a + b; mean, centred variance (two-pass, sequential);
 *              y = (v - mean) * (1/sqrtf(var + eps)) * gamma + beta
 *   concat     Y[r][i*c + j] = Z_i[r][j]
 * Every function is batched over `batch` instances with per-operand instance
 * strides in elements (0 = shared operand). OpenMP spreads instances x rows
 * over the host cores for the CPU baseline.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define AT(p, s, b) ((p) + (int64_t)(b) * (s))

void or_gemm(const float* A, int64_t sA, const float* B, int64_t sB, float* C, int64_t sC, int M, int N, int K,
             int nt, int relu, int batch) {
  int64_t rows = (int64_t)batch * M;
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < rows; ++r) {
    int b = (int)(r / M), i = (int)(r % M);
    const float* a = AT(A, sA, b) + (int64_t)i * K;
    const float* bm = AT(B, sB, b);
    float* c = AT(C, sC, b) + (int64_t)i * N;
    if (!nt) {
      for (int j = 0; j < N; ++j) c[j] = 0.0f;
      for (int k = 0; k < K; ++k) {
        const float av = a[k];
        const float* brow = bm + (int64_t)k * N;
        for (int j = 0; j < N; ++j) c[j] = c[j] + av * brow[j];
      }
    } else {
      for (int j = 0; j < N; ++j) {
        const float* brow = bm + (int64_t)j * K;
        float acc = 0.0f;
        for (int k = 0; k < K; ++k) acc = acc + a[k] * brow[k];
        c[j] = acc;
      }
    }
    if (relu)
      for (int j = 0; j < N; ++j) c[j] = c[j] > 0.0f ? c[j] : 0.0f;
  }
}

void or_transpose(const float* A, int64_t sA, float* B, int64_t sB, int R, int Cc, int batch) {
#pragma omp parallel for schedule(static)
  for (int b = 0; b < batch; ++b) {
    const float* a = AT(A, sA, b);
    float* o = AT(B, sB, b);
    for (int r = 0; r < R; ++r)
      for (int c = 0; c < Cc; ++c) o[(int64_t)c * R + r] = a[(int64_t)r * Cc + c];
  }
}

void or_scale(const float* A, int64_t sA, float* B, int64_t sB, int64_t n, float s, int batch) {
#pragma omp parallel for schedule(static)
  for (int b = 0; b < batch; ++b) {
    const float* a = AT(A, sA, b);
    float* o = AT(B, sB, b);
    for (int64_t i = 0; i < n; ++i) o[i] = a[i] * s;
  }
}

void or_add(const float* A, int64_t sA, const float* B, int64_t sB, float* C, int64_t sC, int64_t n, int batch) {
#pragma omp parallel for schedule(static)
  for (int b = 0; b < batch; ++b) {
    const float* a = AT(A, sA, b);
    const float* bb = AT(B, sB, b);
    float* c = AT(C, sC, b);
    for (int64_t i = 0; i < n; ++i) c[i] = a[i] + bb[i];
  }
}

void or_softmax(const float* A, int64_t sA, float* B, int64_t sB, int rows, int cols, float s, int batch) {
  int64_t total = (int64_t)batch * rows;
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < total; ++r) {
    int b = (int)(r / rows), i = (int)(r % rows);
    const float* a = AT(A, sA, b) + (int64_t)i * cols;
    float* o = AT(B, sB, b) + (int64_t)i * cols;
    float m = -INFINITY;
    for (int j = 0; j < cols; ++j) {
      float x = a[j] * s;
      if (x > m) m = x;
    }
    float sum = 0.0f;
    for (int j = 0; j < cols; ++j) {
      float e = expf(a[j] * s - m);
      o[j] = e;
      sum = sum + e;
    }
    for (int j = 0; j < cols; ++j) o[j] = o[j] / sum;
  }
}

void or_add_layernorm(const float* A, int64_t sA, const float* B, int64_t sB, const float* G, int64_t sG,
                      const float* Be, int64_t sBe, float* Y, int64_t sY, int rows, int cols, float eps, int batch) {
  int64_t total = (int64_t)batch * rows;
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < total; ++r) {
    int b = (int)(r / rows), i = (int)(r % rows);
    const float* a = AT(A, sA, b) + (int64_t)i * cols;
    const float* bb = AT(B, sB, b) + (int64_t)i * cols;
    const float* g = AT(G, sG, b);
    const float* be = AT(Be, sBe, b);
    float* y = AT(Y, sY, b) + (int64_t)i * cols;
    float sum = 0.0f;
    for (int j = 0; j < cols; ++j) {
      y[j] = a[j] + bb[j];
      sum = sum + y[j];
    }
    float mean = sum / (float)cols;
    float q = 0.0f;
    for (int j = 0; j < cols; ++j) {
      float d = y[j] - mean;
      q = q + d * d;
    }
    float var = q / (float)cols;
    float rstd = 1.0f / sqrtf(var + eps);
    for (int j = 0; j < cols; ++j) y[j] = (y[j] - mean) * rstd * g[j] + be[j];
  }
}

void or_concat(const float* const* Z, const int64_t* sZ, int count, float* Y, int64_t sY, int rows, int cols_each,
               int batch) {
#pragma omp parallel for schedule(static)
  for (int b = 0; b < batch; ++b) {
    float* y = AT(Y, sY, b);
    for (int i = 0; i < count; ++i) {
      const float* z = AT(Z[i], sZ[i], b);
      for (int r = 0; r < rows; ++r)
        memcpy(y + (int64_t)r * cols_each * count + (int64_t)i * cols_each, z + (int64_t)r * cols_each,
               sizeof(float) * (size_t)cols_each);
    }
  }
}

/* fp64-accumulated GEMM ("truth" for error-headroom reporting). */
void or_gemm_f64(const float* A, int64_t sA, const float* B, int64_t sB, double* C, int64_t sC, int M, int N, int K,
                 int nt, int batch) {
  int64_t rows = (int64_t)batch * M;
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < rows; ++r) {
    int b = (int)(r / M), i = (int)(r % M);
    const float* a = AT(A, sA, b) + (int64_t)i * K;
    const float* bm = AT(B, sB, b);
    double* c = C + (int64_t)b * sC + (int64_t)i * N;
    for (int j = 0; j < N; ++j) c[j] = 0.0;
    for (int k = 0; k < K; ++k)
      for (int j = 0; j < N; ++j)
        c[j] += (double)a[k] * (double)(nt ? bm[(int64_t)j * K + k] : bm[(int64_t)k * N + j]);
  }
}

int or_max_threads(void) {
#ifdef _OPENMP
  extern int omp_get_max_threads(void);
  return omp_get_max_threads();
#else
  return 1;
#endif
}
