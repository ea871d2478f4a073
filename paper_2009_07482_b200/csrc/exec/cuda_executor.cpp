// hetsim::CudaExecutor (include/hetsim/cuda_executor.hpp): the public C++
// executor for Alg. 1's dispatch entry point, backed by a dynamic-mode Engine.
#include "hetsim/cuda_executor.hpp"

#include <string>

#include "engine.hpp"
#include "hetsim/errors.hpp"

namespace hetsim {

CudaExecutor::CudaExecutor(const DagSpec& g, const CudaExecutorOptions& opts) {
  EngineConfig cfg;
  cfg.spec_text = serialize(g);
  cfg.params = g.params;
  cfg.gpu = opts.gpu;
  cfg.graph_mode = false;
  cfg.batch = opts.batch;
  cfg.slots = 1;
  cfg.deterministic = opts.deterministic;
  const std::string m = opts.math ? opts.math : "tf32x3";
  if (m == "tf32x3") cfg.math = HS_MATH_TF32X3;
  else if (m == "tf32") cfg.math = HS_MATH_TF32;
  else if (m == "bf16x3") cfg.math = HS_MATH_BF16X3;
  else if (m == "simt") cfg.math = HS_MATH_FP32_SIMT;
  else fail(Errc::invalid_param, "math must be tf32x3|tf32|bf16x3|simt");
  engine_ = std::make_unique<Engine>(std::move(cfg));
}

CudaExecutor::~CudaExecutor() = default;

void CudaExecutor::bind(int kernel, int pos, void* ptr, int64_t stride_bytes, int64_t count, bool on_device) {
  engine_->bind(kernel, pos, ptr, stride_bytes, count, on_device);
}

void CudaExecutor::begin(int64_t first, int64_t n) { engine_->ext_begin(first, n); }

void CudaExecutor::dispatch(const TaskComponent& t, const CommandQueueStructure& q) { engine_->ext_dispatch(t, q); }

Completion CudaExecutor::wait_next() { return engine_->ext_wait(); }

int64_t CudaExecutor::end() { return engine_->ext_end(); }

}  // namespace hetsim
