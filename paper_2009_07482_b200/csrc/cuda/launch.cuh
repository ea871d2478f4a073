// Kernel launch with programmatic dependent launch (PDL) for every DAG node kernel.
//
// Consecutive node kernels on one CUDA stream (one command queue of a component)
// are launched with cudaLaunchAttributeProgrammaticStreamSerialization: the next
// kernel's CTAs may start as soon as every CTA of the previous one has executed
// griddepcontrol.launch_dependents, run their prologue (barrier init, TMEM
// allocation, tensor-map prefetch) and then block in griddepcontrol.wait, which
// returns once the previous grid has completed and its memory is visible. Every
// node kernel calls pdl_launch_dependents() + pdl_wait() after its prologue and
// before its first global-memory access, so data dependencies (and buffer reuse
// by the liveness arena) are exactly those of a plain launch. Stream capture turns
// the attribute into programmatic graph edges. HS_PDL=0 in the environment
// launches without it (A/B).
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>

#define HS_TRY(x)                   \
  do {                              \
    const cudaError_t e_ = (x);     \
    if (e_ != cudaSuccess) return e_; \
  } while (0)

namespace hs {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("HS_PDL");
    return !(v && std::strcmp(v, "0") == 0);
  }();
  return on;
}

// cudaLaunchKernelEx with PDL (when enabled) and an optional 1-D cluster.
template <typename... KArgs, typename... Args>
cudaError_t launch_node(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, int cluster,
                        Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  unsigned n = 0;
  if (cluster > 1) {
    at[n].id = cudaLaunchAttributeClusterDimension;
    at[n].val.clusterDim.x = unsigned(cluster);
    at[n].val.clusterDim.y = 1;
    at[n].val.clusterDim.z = 1;
    ++n;
  }
  if (pdl_enabled()) {
    at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  cfg.attrs = at;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace hs
