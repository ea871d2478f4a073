// Probe: how tcgen05.mma kind::tf32 reads an fp32 operand whose low 13 mantissa bits are
// not zero. A row m holds s * (1 + m * 2^-14) (tf32 keeps 10 mantissa bits, so the low part
// of m * 2^-14 sits below the tf32 ulp); B rows are +1 / -1 (exact). D[m][n] / 8 over K = 8 is
// the value the tensor core used for A[m]: compared with round-toward-zero and round-to-nearest.
// Operand A from shared memory (ss) and from TMEM (ts).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/tf32_trunc profiles/tf32_trunc_probe.cu -lcuda
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>

#include "../paper_2009_07482_b200/csrc/cuda/tc_common.cuh"

using namespace hs::tc;

__device__ float a_val(int m, int sign) { return sign * (1.0f + float(m) * 0x1p-14f); }

template <bool kTs>
__global__ void __launch_bounds__(128, 1) probe(float* out, int sign) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t sA = base, sB = base + 16384, bar = base + 32768, slot = bar + 8;
  const int warp = threadIdx.x >> 5, t = threadIdx.x;
  // A: 128 rows x 32 fp32 (SW128 rows; every element of a row equal, so the swizzle is moot)
  for (int k = 0; k < 32; ++k) sts32(sA + t * 128 + k * 4, a_val(t, sign));
  // B: 64 rows, row n = +1 (n even) / -1 (n odd)
  if (t < 64)
    for (int k = 0; k < 32; ++k) sts32(sB + t * 128 + k * 4, (t & 1) ? -1.0f : 1.0f);
  if (t == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(slot), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem_raw + (slot - smem_u32(smem_raw)));
  const uint32_t lane_base = uint32_t(warp * 32) << 16;
  if constexpr (kTs) {  // A (raw fp32 bits) into TMEM columns [128, 136)
    uint32_t v[16];
    for (int i = 0; i < 16; ++i) v[i] = __float_as_uint(a_val(t, sign));
    tmem_st16(tmem + lane_base + 128u, v);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    tc_fence_before();
  }
  __syncthreads();
  tc_fence_after();
  constexpr uint32_t idesc = instr_desc_tf32(64);
  if (warp == 1 && elect_one()) {
    if constexpr (kTs) mma_tf32_ts(tmem, tmem + 128u, smem_desc(sB), idesc, 0u);
    else mma_tf32(tmem, smem_desc(sA), smem_desc(sB), idesc, 0u);
    mma_commit(bar);
  }
  mbar_wait(bar, 0);
  tc_fence_after();
  uint32_t r[32];
  tmem_ld32(tmem + lane_base, r);
  tmem_ld_wait(r);
  out[t * 2 + 0] = __uint_as_float(r[0]) / 8.0f;
  out[t * 2 + 1] = __uint_as_float(r[1]) / 8.0f;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
  }
}

static float rz(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  u &= 0xFFFFE000u;
  memcpy(&x, &u, 4);
  return x;
}
static float rne(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  const uint32_t lsb = (u >> 13) & 1u;
  u = (u + 0xFFFu + lsb) & 0xFFFFE000u;
  memcpy(&x, &u, 4);
  return x;
}
static float rna(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  u = (u + 0x1000u) & 0xFFFFE000u;
  memcpy(&x, &u, 4);
  return x;
}

template <bool kTs>
void run(const char* name, float* d, int sign) {
  auto k = probe<kTs>;
  const int smem = 32768 + 2048;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<<<1, 128, smem>>>(d, sign);
  cudaError_t e = cudaDeviceSynchronize();
  float h[256];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  int n_rz = 0, n_rne = 0, n_rna = 0, n_exact = 0, n_neg = 0;
  for (int m = 0; m < 128; ++m) {
    const float a = sign * (1.0f + float(m) * 0x1p-14f);
    n_rz += h[2 * m] == rz(a);
    n_rne += h[2 * m] == rne(a);
    n_rna += h[2 * m] == rna(a);
    n_exact += h[2 * m] == a;
    n_neg += h[2 * m + 1] == -h[2 * m];
  }
  printf("%s sign=%+d: of 128 rows the tensor core used  rz %d  rne %d  rna %d  exact fp32 %d  (B=-1 column symmetric %d) %s\n",
         name, sign, n_rz, n_rne, n_rna, n_exact, n_neg, e ? cudaGetErrorString(e) : "");
  printf("  rows 0..20 used/8:");
  for (int m = 0; m < 21; ++m) printf(" %.7f", h[2 * m]);
  printf("\n");
}

int main() {
  float* d;
  cudaMalloc(&d, 1024);
  for (int s : {1, -1}) {
    run<false>("A from smem (ss)", d, s);
    run<true>("A from TMEM (ts)", d, s);
  }
  return 0;
}
