// hetsim-b200 — the B200 executor behind the scheduler's dispatch entry point.
//
// The reference's dispatch(T, Q*) submits every queue of a component's command
// queue structure at the current clock and locks the device until the
// component's callback-marked commands complete (the paper's
// clFlush per queue). Its downstream is platform_sim
// (SPEC.md:386). CudaExecutor replaces that simulator with the B200:
//   queue i of T on logical device d  -> a CUDA stream
//   E_Q pair / inter edge             -> CUDA events (stream waits, no host sync)
//   ndrange                           -> an sm_100a kernel over the bound instances
//   isolated write / read             -> H2D / D2H on the copy engines
//   callback mark                     -> cudaLaunchHostFunc -> wait_next()
// so a C++ caller runs Alg. 1 on real hardware exactly as it would on the
// simulator:
//
//   hetsim::DagSpec g = hetsim::parse_spec(text, params);
//   hetsim::CudaExecutor ex(g, {.batch = 64});
//   ex.bind(kernel, pos, host_ptr, stride_bytes, count);   // every isolated buffer
//   ex.begin(first, n);                                    // instances of this run
//   auto r = hetsim::run_schedule(g, hetsim::Platform::from_spec(g), {}, hetsim::Policy::clustering, ex);
//   int64_t ns = ex.end();                                 // outputs are in the bound memory
//
// One run_schedule call covers n <= batch instances: every ndrange is one kernel
// launch over all n (instance-batched node launches).
#pragma once

#include <cstdint>
#include <memory>

#include "hetsim/scheduler.hpp"
#include "hetsim/spec_model.hpp"

namespace hetsim {

class Engine;

struct CudaExecutorOptions {
  int gpu = 0;
  int batch = 1;               // instances per kernel launch (max n of begin())
  const char* math = "tf32x3"; // tf32x3 | tf32 | bf16x3 | simt
  bool deterministic = false;  // no split-K: bit-reproducible single-instance GEMMs
};

class CudaExecutor : public Executor {
 public:
  explicit CudaExecutor(const DagSpec& g, const CudaExecutorOptions& opts = {});
  ~CudaExecutor() override;
  CudaExecutor(const CudaExecutor&) = delete;
  CudaExecutor& operator=(const CudaExecutor&) = delete;

  /// Isolated input/output buffer (kernel, pos) -> memory holding `count`
  /// instances `stride_bytes` apart (stride 0: one copy shared by all instances,
  /// uploaded once). on_device: ptr is device memory on the executor's GPU.
  void bind(int kernel, int pos, void* ptr, int64_t stride_bytes, int64_t count, bool on_device = false);
  /// Start a run over instances [first, first + n), n <= batch (InvalidParam).
  void begin(int64_t first, int64_t n);
  void dispatch(const TaskComponent& t, const CommandQueueStructure& q) override;
  Completion wait_next() override;
  /// Wait for every issued command; returns the device time of the run in ns.
  int64_t end();

 private:
  std::unique_ptr<Engine> engine_;
};

}  // namespace hetsim
