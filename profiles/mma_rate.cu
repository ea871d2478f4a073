// Probe: issue rate / execution rate of single-CTA tcgen05.mma (cta_group::1, kind::tf32
// and kind::f16) by shape and operand source: A from TMEM (ts) or shared memory (ss),
// N = 64..256, M = 128, with and without the disable-output-lane mask operand.
// One CTA per SM; CTA 0 reports cycles per MMA (issue loop and until the commit lands).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/mma_rate profiles/mma_rate.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../paper_2009_07482_b200/csrc/cuda/tc_common.cuh"

using namespace hs::tc;

constexpr int kIters = 512;

template <int kKind, bool kTs, bool kMask>
__device__ __forceinline__ void mma1(uint32_t d, uint32_t a_tmem, uint64_t a_desc, uint64_t b, uint32_t idesc,
                                     uint32_t acc) {
  if constexpr (kTs) {
    if constexpr (kMask) {
      if constexpr (kKind == 0) mma_tf32_ts(d, a_tmem, b, idesc, acc);
      else mma_f16_ts(d, a_tmem, b, idesc, acc);
    } else {
      if constexpr (kKind == 0)
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
            "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
            : "memory");
      else
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
            "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
            : "memory");
    }
  } else {
    if constexpr (kKind == 0)
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
          "l"(a_desc), "l"(b), "r"(idesc), "r"(acc)
          : "memory");
    else
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
          "l"(a_desc), "l"(b), "r"(idesc), "r"(acc)
          : "memory");
  }
}

template <int kKind, bool kTs, bool kMask, int N>
__global__ void __launch_bounds__(128, 1) rate(long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t sA = base, sB = base + 65536, bar = base + 2 * 65536, slot = bar + 8;
  const int warp = threadIdx.x >> 5;
  // zero operands (rate does not depend on values)
  for (uint32_t o = threadIdx.x * 16; o < 2 * 65536; o += 128 * 16) sts128(base + o, make_float4(0, 0, 0, 0));
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(slot), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem_raw + (slot - smem_u32(smem_raw)));
  constexpr uint32_t idesc = kKind == 0 ? instr_desc_tf32(N) : instr_desc_bf16(N);
  long long t0 = 0, t1 = 0, t2 = 0;
  if (warp == 1 && elect_one()) {
    t0 = clock64();
    for (int i = 0; i < kIters; ++i) {
      const uint32_t kk = uint32_t(i & 3);
      mma1<kKind, kTs, kMask>(tmem, tmem + 384u + kk * 8u, smem_desc(sA + kk * 32u), smem_desc(sB + kk * 32u), idesc,
                               i ? 1u : 0u);
    }
    t1 = clock64();
    mma_commit(bar);
    mbar_wait(bar, 0);
    t2 = clock64();
    if (blockIdx.x == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

template <int kKind, bool kTs, bool kMask, int N>
void run(const char* name, long long* d) {
  auto k = rate<kKind, kTs, kMask, N>;
  const int smem = 2 * 65536 + 2048;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int rep = 0; rep < 3; ++rep) k<<<148, 128, smem>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[2];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const double flop = 2.0 * 128 * N * (kKind == 0 ? 8 : 16);
  printf("%-28s N=%3d  issue %6.1f cyc/mma  complete %6.1f cyc/mma  (%5.0f flop/cyc/SM) %s\n", name, N,
         double(h[0]) / kIters, double(h[1]) / kIters, flop * kIters / double(h[1]), e ? cudaGetErrorString(e) : "");
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  run<0, true, true, 64>("tf32 ts mask", d);
  run<0, true, true, 128>("tf32 ts mask", d);
  run<0, true, true, 192>("tf32 ts mask", d);
  run<0, true, true, 256>("tf32 ts mask", d);
  run<0, true, false, 64>("tf32 ts", d);
  run<0, true, false, 128>("tf32 ts", d);
  run<0, true, false, 256>("tf32 ts", d);
  run<0, false, false, 64>("tf32 ss", d);
  run<0, false, false, 128>("tf32 ss", d);
  run<0, false, false, 256>("tf32 ss", d);
  run<1, true, false, 64>("bf16 ts", d);
  run<1, true, false, 128>("bf16 ts", d);
  run<1, true, false, 256>("bf16 ts", d);
  run<1, false, false, 64>("bf16 ss", d);
  run<1, false, false, 256>("bf16 ss", d);
  return 0;
}
