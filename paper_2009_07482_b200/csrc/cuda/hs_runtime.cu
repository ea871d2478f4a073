// The thin C ABI between the C++ executor and CUDA (include/hetsim_c.h §2).
//
// Every entry point returns 0 or a non-zero status and records a
// thread-local "<Errc>: message" for hs_last_error(); no C++ exception
// crosses it. Node kernels are dispatched by op id to the sm_100a
// implementations in kernels_mem.cu / gemm_tc.cu / gemm_simt.cu.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstring>
#include <string>

#include "hetsim_c.h"
#include "kernels.cuh"

struct hs_ctx {
  int gpu;
};
struct hs_stream {
  int gpu;
  cudaStream_t s;
};
struct hs_event {
  int gpu;
  cudaEvent_t e;
};
struct hs_graph {
  int gpu;
  cudaGraph_t g;
  cudaGraphExec_t exec;
};

namespace {

thread_local std::string t_error;
thread_local int t_errc = -1;
thread_local int t_device = -1;
std::atomic<int64_t> g_launches{0};

// Errc ordinals (include/hetsim/errors.hpp): invalid_param = 10, device_error = 19.
constexpr int kErrcInvalidParam = 10;
constexpr int kErrcDeviceError = 19;

int set_error(int status, int errc, const std::string& msg) {
  t_errc = errc;
  t_error = (errc == kErrcDeviceError ? "DeviceError: " : "InvalidParam: ") + msg;
  return status;
}

int check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return HS_OK;
  return set_error(HS_ERR_CUDA, kErrcDeviceError, std::string(what) + ": " + cudaGetErrorString(e));
}

int invalid(const char* what) { return set_error(HS_ERR_INVALID, kErrcInvalidParam, what); }

int use_device(int gpu) {
  if (t_device == gpu) return HS_OK;
  int r = check(cudaSetDevice(gpu), "cudaSetDevice");
  if (r == HS_OK) t_device = gpu;
  return r;
}

}  // namespace

extern "C" {

// Private: lets the C++ engine / query layers report through the same slot.
int hs__set_error(int status, int errc, const char* msg) {
  t_errc = errc;
  t_error = msg ? msg : "";
  return status;
}

int hs_memcpy_2d(hs_stream_t s, void* dst, size_t dpitch, const void* src, size_t spitch, size_t width,
                 size_t height, int kind) {
  if (!s) return invalid("null stream");
  static const cudaMemcpyKind kinds[4] = {cudaMemcpyHostToDevice, cudaMemcpyDeviceToHost, cudaMemcpyDeviceToDevice,
                                          cudaMemcpyDefault};
  if (kind < 0 || kind > 3) return invalid("bad copy kind");
  if (height == 0 || width == 0) return HS_OK;
  if (dpitch == width && spitch == width)
    return check(cudaMemcpyAsync(dst, src, width * height, kinds[kind], s->s), "cudaMemcpyAsync");
  return check(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, kinds[kind], s->s), "cudaMemcpy2DAsync");
}

const char* hs_last_error(void) { return t_error.c_str(); }
int hs_last_errc(void) { return t_errc; }
const char* hs_version(void) { return "hetsim-b200 0.1 (sm_100a)"; }

int hs_device_count(int* count) {
  if (!count) return invalid("null count");
  return check(cudaGetDeviceCount(count), "cudaGetDeviceCount");
}

int hs_ctx_create(int gpu, hs_ctx_t* out) {
  if (!out) return invalid("null out");
  int n = 0;
  if (int r = check(cudaGetDeviceCount(&n), "cudaGetDeviceCount")) return r;
  if (gpu < 0 || gpu >= n) return invalid("gpu ordinal out of range");
  if (int r = use_device(gpu)) return r;
  if (int r = check(cudaFree(nullptr), "context init")) return r;
  *out = new hs_ctx{gpu};
  return HS_OK;
}

int hs_ctx_destroy(hs_ctx_t ctx) {
  delete ctx;
  return HS_OK;
}

int hs_ctx_sync(hs_ctx_t ctx) {
  if (!ctx) return invalid("null ctx");
  if (int r = use_device(ctx->gpu)) return r;
  return check(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
}

int hs_stream_create(hs_ctx_t ctx, int priority, hs_stream_t* out) {
  if (!ctx || !out) return invalid("null argument");
  if (int r = use_device(ctx->gpu)) return r;
  cudaStream_t s;
  if (int r = check(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, priority), "cudaStreamCreate")) return r;
  *out = new hs_stream{ctx->gpu, s};
  return HS_OK;
}

int hs_stream_destroy(hs_stream_t s) {
  if (!s) return HS_OK;
  use_device(s->gpu);
  cudaStreamDestroy(s->s);
  delete s;
  return HS_OK;
}

int hs_stream_sync(hs_stream_t s) {
  if (!s) return invalid("null stream");
  return check(cudaStreamSynchronize(s->s), "cudaStreamSynchronize");
}

int hs_event_create(hs_ctx_t ctx, int timing, hs_event_t* out) {
  if (!ctx || !out) return invalid("null argument");
  if (int r = use_device(ctx->gpu)) return r;
  cudaEvent_t e;
  if (int r = check(cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming), "cudaEventCreate"))
    return r;
  *out = new hs_event{ctx->gpu, e};
  return HS_OK;
}

int hs_event_destroy(hs_event_t e) {
  if (!e) return HS_OK;
  use_device(e->gpu);
  cudaEventDestroy(e->e);
  delete e;
  return HS_OK;
}

int hs_event_record(hs_event_t e, hs_stream_t s) {
  if (!e || !s) return invalid("null argument");
  return check(cudaEventRecord(e->e, s->s), "cudaEventRecord");
}

int hs_stream_wait(hs_stream_t s, hs_event_t e) {
  if (!e || !s) return invalid("null argument");
  return check(cudaStreamWaitEvent(s->s, e->e, 0), "cudaStreamWaitEvent");
}

int hs_event_sync(hs_event_t e) {
  if (!e) return invalid("null event");
  return check(cudaEventSynchronize(e->e), "cudaEventSynchronize");
}

int hs_event_elapsed_ns(hs_event_t from, hs_event_t to, int64_t* ns) {
  if (!from || !to || !ns) return invalid("null argument");
  float ms = 0.f;
  if (int r = check(cudaEventElapsedTime(&ms, from->e, to->e), "cudaEventElapsedTime")) return r;
  *ns = int64_t(double(ms) * 1e6);
  return HS_OK;
}

int hs_malloc(hs_ctx_t ctx, size_t bytes, void** out) {
  if (!ctx || !out) return invalid("null argument");
  if (int r = use_device(ctx->gpu)) return r;
  return check(cudaMalloc(out, bytes ? bytes : 16), "cudaMalloc");
}

int hs_free(hs_ctx_t ctx, void* p) {
  if (!ctx) return invalid("null ctx");
  if (!p) return HS_OK;
  if (int r = use_device(ctx->gpu)) return r;
  return check(cudaFree(p), "cudaFree");
}

int hs_host_alloc(size_t bytes, void** out) {
  if (!out) return invalid("null out");
  return check(cudaHostAlloc(out, bytes ? bytes : 16, cudaHostAllocPortable), "cudaHostAlloc");
}
int hs_host_free(void* p) { return p ? check(cudaFreeHost(p), "cudaFreeHost") : HS_OK; }
int hs_host_pin(void* p, size_t bytes) {
  if (!p) return invalid("null pointer");
  return check(cudaHostRegister(p, bytes, cudaHostRegisterPortable), "cudaHostRegister");
}
int hs_host_unpin(void* p) { return p ? check(cudaHostUnregister(p), "cudaHostUnregister") : HS_OK; }

int hs_memcpy_h2d(hs_stream_t s, void* dst, const void* src, size_t bytes) {
  if (!s) return invalid("null stream");
  return check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s->s), "cudaMemcpyAsync H2D");
}
int hs_memcpy_d2h(hs_stream_t s, void* dst, const void* src, size_t bytes) {
  if (!s) return invalid("null stream");
  return check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s->s), "cudaMemcpyAsync D2H");
}
int hs_memcpy_d2d(hs_stream_t s, void* dst, const void* src, size_t bytes) {
  if (!s) return invalid("null stream");
  return check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s->s), "cudaMemcpyAsync D2D");
}
int hs_memcpy_peer(hs_stream_t s, void* dst, int dst_gpu, const void* src, int src_gpu, size_t bytes) {
  if (!s) return invalid("null stream");
  if (int r = use_device(s->gpu)) return r;
  if (dst_gpu == src_gpu)  // one GPU (e.g. two memory domains of a 1-GPU engine): a device copy
    return check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s->s), "cudaMemcpyAsync");
  return check(cudaMemcpyPeerAsync(dst, dst_gpu, src, src_gpu, bytes, s->s), "cudaMemcpyPeerAsync");
}

int hs_ctx_enable_peer(hs_ctx_t a, hs_ctx_t b) {
  if (!a || !b) return invalid("null context");
  if (a->gpu == b->gpu) return HS_OK;
  int can = 0;
  if (int r = check(cudaDeviceCanAccessPeer(&can, a->gpu, b->gpu), "cudaDeviceCanAccessPeer")) return r;
  if (!can) return HS_OK;
  if (int r = use_device(a->gpu)) return r;
  cudaError_t e = cudaDeviceEnablePeerAccess(b->gpu, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return HS_OK;
  }
  return check(e, "cudaDeviceEnablePeerAccess");
}
int hs_memset(hs_stream_t s, void* dst, int value, size_t bytes) {
  if (!s) return invalid("null stream");
  return check(cudaMemsetAsync(dst, value, bytes, s->s), "cudaMemsetAsync");
}

int hs_op_from_name(const char* name) {
  static const char* kNames[HS_OP_COUNT] = {"gemm",    "gemm_nt", "gemm_relu", "transpose",   "scale",
                                             "softmax", "add",     "add_layernorm", "concat",
                                             "attn_head", nullptr /* HS_OP_HEAD: engine rewrite only */};
  if (!name) return -1;
  for (int i = 0; i < HS_OP_COUNT; ++i)
    if (kNames[i] && std::strcmp(name, kNames[i]) == 0) return i;
  return -1;
}

int hs_launch(hs_stream_t st, int op, const hs_op_args* a, int math, int batch) {
  if (!st || !a) return invalid("null argument");
  if (batch < 1) return invalid("batch must be >= 1");
  if (int r = use_device(st->gpu)) return r;
  const cudaStream_t s = st->s;
  auto in = [&](int i) { return static_cast<const float*>(a->in[i]); };
  auto out = static_cast<float*>(a->out);
  cudaError_t e = cudaSuccess;
  switch (op) {
    case HS_OP_GEMM:
    case HS_OP_GEMM_NT:
    case HS_OP_GEMM_RELU: {
      if (a->n_in < 2) return invalid("gemm needs two inputs");
      hs::GemmArgs g{in(0), a->in_stride[0], in(1), a->in_stride[1], out, a->out_stride,
                     int(a->dims[0]), int(a->dims[1]), int(a->dims[2]), batch,
                     op == HS_OP_GEMM_NT ? hs::GemmLayout::nt : hs::GemmLayout::nn, op == HS_OP_GEMM_RELU,
                     math == HS_MATH_FP32_SIMT ? nullptr : static_cast<const float*>(a->aux)};
      if (a->out_ld < 0 || (a->out_ld > 0 && a->out_ld < a->dims[1])) return invalid("gemm out_ld < N");
      if (a->epilogue != HS_EPI_NONE && a->epilogue != HS_EPI_SOFTMAX) return invalid("unknown GEMM epilogue");
      g.ldc = a->out_ld;
      g.deterministic = (a->flags & HS_FLAG_DETERMINISTIC) != 0;
      if (a->epilogue == HS_EPI_SOFTMAX) {
        if (math == HS_MATH_FP32_SIMT || op == HS_OP_GEMM_RELU || a->n_out > 1 || a->dims[1] > 128)
          return invalid("softmax epilogue needs tcgen05 math, a plain GEMM and N <= 128");
        g.softmax = 1;
        g.escale = a->fparam[0];
      }
      // BF16X3 applies to GEMMs whose B arrives pre-split (bf16 planes); the rest run TF32X3.
      g.bf16 = (math == HS_MATH_BF16X3 && a->aux) ? 1 : 0;
      if (g.bf16 && (g.K % 8) && a->n_out <= 1) {
        // bf16 planes need 16-byte rows (K % 8 == 0) for TMA: split B in-kernel instead (TF32X3)
        g.bf16 = 0;
        g.Bplanes = nullptr;
      }
      if (a->n_out > 1) {
        // grouped launch of sibling GEMMs (tcgen05 only; the caller checked eligibility)
        if (a->n_out > 4 || !a->aux || math == HS_MATH_FP32_SIMT) return invalid("bad grouped GEMM launch");
        g.n_out = a->n_out;
        g.N = int(a->dims[1]) * a->n_out;
        for (int i = 0; i < a->n_out; ++i) {
          g.Cs[i] = static_cast<float*>(a->outs[i]);
          g.sCs[i] = a->out_strides[i];
        }
        g.C = g.Cs[0];
        g.sC = g.sCs[0];
        if (!hs::gemm_tcgen05_supported(g)) return invalid("grouped GEMM shape not supported");
        e = hs::gemm_tcgen05(g, math == HS_MATH_TF32 ? 1 : 3, s);
      } else if (math == HS_MATH_FP32_SIMT || !hs::gemm_tcgen05_supported(g)) {
        if (g.softmax) return invalid("softmax epilogue: GEMM shape not supported by the tcgen05 path");
        e = hs::gemm_simt(g, s);
      } else {
        e = hs::gemm_tcgen05(g, math == HS_MATH_TF32 ? 1 : 3, s);
      }
      break;
    }
    case HS_OP_TRANSPOSE:
      e = hs::transpose(in(0), a->in_stride[0], out, a->out_stride, int(a->dims[0]), int(a->dims[1]), batch, s);
      break;
    case HS_OP_SCALE:
      e = hs::scale(in(0), a->in_stride[0], out, a->out_stride, a->dims[0], a->fparam[0], batch, s);
      break;
    case HS_OP_SOFTMAX:
      e = hs::softmax(in(0), a->in_stride[0], out, a->out_stride, int(a->dims[0]), int(a->dims[1]), a->fparam[0],
                      batch, s);
      break;
    case HS_OP_ADD:
      if (a->n_in < 2) return invalid("add needs two inputs");
      e = hs::add(in(0), a->in_stride[0], in(1), a->in_stride[1], out, a->out_stride, a->dims[0], batch, s);
      break;
    case HS_OP_ADD_LN:
      if (a->n_in < 4) return invalid("add_layernorm needs four inputs");
      e = hs::add_layernorm(in(0), a->in_stride[0], in(1), a->in_stride[1], in(2), a->in_stride[2], in(3),
                            a->in_stride[3], out, a->out_stride, int(a->dims[0]), int(a->dims[1]), a->fparam[1], batch,
                            s);
      break;
    case HS_OP_CONCAT: {
      const float* z[HS_MAX_INPUTS];
      for (int i = 0; i < a->n_in; ++i) z[i] = in(i);
      e = hs::concat(z, a->in_stride, a->n_in, out, a->out_stride, int(a->dims[0]), int(a->dims[1]), batch, s);
      break;
    }
    case HS_OP_ATTN_HEAD: {
      if (a->n_in < 4 || !a->aux) return invalid("attn_head needs {Q, K, V, W} and pre-split W planes (aux)");
      if (math == HS_MATH_FP32_SIMT) return invalid("attn_head runs on the tensor cores only");
      hs::AttnArgs t{in(0), a->in_stride[0], in(1), a->in_stride[1], in(2), a->in_stride[2], a->aux,
                     out,   a->out_stride,   a->out_ld, int(a->dims[0]), int(a->dims[1]), int(a->dims[2]),
                     batch, a->fparam[0]};
      if (!hs::attn_head_supported(t)) return invalid("attn_head: needs S <= 128, dk = dw = 64, 16-byte alignment");
      e = hs::attn_head(t, math == HS_MATH_TF32 ? 1 : 3, s);
      break;
    }
    case HS_OP_HEAD: {
      if (a->n_in < 2 || !a->aux || !a->in[1]) return invalid("head needs {X, Wh planes} and Wqkv planes (aux)");
      if (math != HS_MATH_TF32X3 && math != HS_MATH_TF32) return invalid("head runs in TF32X3 / TF32 only");
      hs::HeadArgs h{in(0), a->in_stride[0], a->aux, a->in[1], out, a->out_stride, a->out_ld,
                     int(a->dims[0]), int(a->dims[1]), int(a->dims[2]), batch, a->fparam[0]};
      if (!hs::head_fused_supported(h)) return invalid("head: needs S <= 128, D % 32 == 0, dk = 64, 16-byte alignment");
      e = hs::head_fused(h, math == HS_MATH_TF32 ? 1 : 3, s);
      break;
    }
    default:
      return invalid("unknown op");
  }
  if (e != cudaSuccess) return check(e, "kernel launch");
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return HS_OK;
}

int64_t hs_launch_count(void) { return g_launches.load(); }

int hs_gemm_split_weights(hs_stream_t st, const void* B, int transposed, int64_t N, int64_t K, void* planes) {
  return hs_gemm_split_weights_strided(st, B, transposed, N, K, planes, N * K);
}

int hs_gemm_split_weights_strided(hs_stream_t st, const void* B, int transposed, int64_t N, int64_t K, void* planes,
                                  int64_t plane_stride) {
  return hs_gemm_split_weights_ex(st, B, transposed, N, K, planes, plane_stride, 0);
}

int hs_gemm_split_weights_ex(hs_stream_t st, const void* B, int transposed, int64_t N, int64_t K, void* planes,
                             int64_t plane_stride, int format) {
  if (!st || !B || !planes) return invalid("null argument");
  if (format != 0 && format != 1) return invalid("format must be 0 (tf32) or 1 (bf16)");
  if (N < 1 || K < 1 || N > (1 << 30) || K > (1 << 30)) return invalid("bad weight shape");
  if (plane_stride < N * K) return invalid("plane stride smaller than one plane");
  if (int r = use_device(st->gpu)) return r;
  cudaError_t e = hs::gemm_split_weights(static_cast<const float*>(B), transposed ? hs::GemmLayout::nt : hs::GemmLayout::nn,
                                         int(N), int(K), planes, plane_stride, st->s, format == 1);
  if (e != cudaSuccess) return check(e, "split weights");
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return HS_OK;
}

int hs_host_callback(hs_stream_t s, void (*fn)(void*), void* user) {
  if (!s || !fn) return invalid("null argument");
  return check(cudaLaunchHostFunc(s->s, fn, user), "cudaLaunchHostFunc");
}

int hs_capture_begin(hs_stream_t s) {
  if (!s) return invalid("null stream");
  if (int r = use_device(s->gpu)) return r;
  return check(cudaStreamBeginCapture(s->s, cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
}

int hs_capture_end(hs_stream_t s, hs_graph_t* out) {
  if (!s || !out) return invalid("null argument");
  cudaGraph_t g = nullptr;
  if (int r = check(cudaStreamEndCapture(s->s, &g), "cudaStreamEndCapture")) return r;
  cudaGraphExec_t exec = nullptr;
  if (int r = check(cudaGraphInstantiate(&exec, g, 0), "cudaGraphInstantiate")) {
    cudaGraphDestroy(g);
    return r;
  }
  *out = new hs_graph{s->gpu, g, exec};
  return HS_OK;
}

int hs_graph_launch(hs_graph_t g, hs_stream_t s) {
  if (!g || !s) return invalid("null argument");
  return check(cudaGraphLaunch(g->exec, s->s), "cudaGraphLaunch");
}

int hs_graph_destroy(hs_graph_t g) {
  if (!g) return HS_OK;
  use_device(g->gpu);
  cudaGraphExecDestroy(g->exec);
  cudaGraphDestroy(g->g);
  delete g;
  return HS_OK;
}

}  // extern "C"
