/*
 * hetsim-b200 C ABI.
 *
 * Three layers, all plain C (no C++/torch types):
 *
 *  1. hs_query        — JSON-in/JSON-out access to the host C++ API
 *                       (parse_spec, derive_components, classify_edges,
 *                       ready_components, bottom_level_ranks, setup_cq,
 *                       run_schedule). Replaces direct calls into the
 *                       reference's C++ library (proj/include/hetsim/ headers).
 *
 *  2. hs_* CUDA layer — the thin layer the C++ executor calls for every device
 *                       action. One CUDA stream per command
 *                       queue, events for E_Q and inter-component edges,
 *                       copies on the copy engines, sm_100a node kernels,
 *                       host callbacks, graph capture. This is what the
 *                       reference's simulator (`dispatch` -> platform_sim,
 *                       SPEC.md:342-349 / 386-440) is replaced by.
 *
 *  3. hs_engine       — the dispatch entry point as a whole: a DAG template
 *                       bound to host buffers and executed on one GPU for a
 *                       stream of instances (dynamic Alg. 1 or captured graph).
 *
 * Conventions: every int-returning function returns 0 on success; non-zero
 * means failure and hs_last_error() (thread-local) holds "<Errc>: message".
 * No C++ exception crosses this boundary.
 */
#ifndef HETSIM_C_H_
#define HETSIM_C_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------- status */
#define HS_OK 0
#define HS_ERR_INVALID 1 /* bad argument / input error (exit code 2 class)  */
#define HS_ERR_CUDA 2    /* CUDA runtime / driver failure (DeviceError)      */
#define HS_ERR_RUNTIME 3 /* scheduling runtime error (exit code 1 class)     */

const char* hs_last_error(void);
/* hetsim::Errc ordinal of the last failure on this thread, -1 if none. */
int hs_last_errc(void);
const char* hs_version(void);

/* ------------------------------------------------------ 1. host queries */
/* Returns a malloc'd JSON document {"ok":true,...} or {"ok":false,"errc":..}.
 * Never NULL. Free with hs_free_string. */
char* hs_query(const char* request_json);
void hs_free_string(char* s);

/* ------------------------------------------------------ 2. CUDA layer  */
typedef struct hs_ctx* hs_ctx_t;
typedef struct hs_stream* hs_stream_t;
typedef struct hs_event* hs_event_t;
typedef struct hs_graph* hs_graph_t;

int hs_device_count(int* count);
int hs_ctx_create(int gpu_ordinal, hs_ctx_t* out);
int hs_ctx_destroy(hs_ctx_t ctx);
int hs_ctx_sync(hs_ctx_t ctx);

int hs_stream_create(hs_ctx_t ctx, int priority, hs_stream_t* out);
int hs_stream_destroy(hs_stream_t s);
int hs_stream_sync(hs_stream_t s);

int hs_event_create(hs_ctx_t ctx, int timing, hs_event_t* out); /* timing=0 for E_Q deps */
int hs_event_destroy(hs_event_t e);
int hs_event_record(hs_event_t e, hs_stream_t s);
int hs_stream_wait(hs_stream_t s, hs_event_t e);
int hs_event_sync(hs_event_t e);
int hs_event_elapsed_ns(hs_event_t from, hs_event_t to, int64_t* ns);

int hs_malloc(hs_ctx_t ctx, size_t bytes, void** out);
int hs_free(hs_ctx_t ctx, void* p);
int hs_host_alloc(size_t bytes, void** out); /* pinned */
int hs_host_free(void* p);
int hs_host_pin(void* p, size_t bytes);
int hs_host_unpin(void* p);

int hs_memcpy_h2d(hs_stream_t s, void* dst, const void* src, size_t bytes);
int hs_memcpy_d2h(hs_stream_t s, void* dst, const void* src, size_t bytes);
int hs_memcpy_d2d(hs_stream_t s, void* dst, const void* src, size_t bytes);
int hs_memcpy_peer(hs_stream_t s, void* dst, int dst_gpu, const void* src, int src_gpu, size_t bytes);
/* Let kernels and copies of ctx `a`'s GPU reach ctx `b`'s memory directly over
 * NVLink (cudaDeviceEnablePeerAccess); a no-op for the same GPU or when the
 * pair has no peer path (peer copies then stage through the host). */
int hs_ctx_enable_peer(hs_ctx_t a, hs_ctx_t b);
int hs_memset(hs_stream_t s, void* dst, int value, size_t bytes);
/* Strided copy of `height` rows of `width` bytes; kind 0=H2D 1=D2H 2=D2D 3=default. */
int hs_memcpy_2d(hs_stream_t s, void* dst, size_t dpitch, const void* src, size_t spitch, size_t width,
                 size_t height, int kind);

/* DAG node operators (kernel "name" in the spec). Argument conventions
 * (buffer positions / var-args) are listed in DESIGN.md §4. */
typedef enum {
  HS_OP_GEMM = 0,      /* C[M,N] = A[M,K] B[K,N]                  */
  HS_OP_GEMM_NT = 1,   /* C[M,N] = A[M,K] B[N,K]^T                */
  HS_OP_GEMM_RELU = 2, /* C = max(0, A B)                         */
  HS_OP_TRANSPOSE = 3, /* B[C,R] = A[R,C]^T                       */
  HS_OP_SCALE = 4,     /* B = A * s                               */
  HS_OP_SOFTMAX = 5,   /* row softmax of (A * s)                  */
  HS_OP_ADD = 6,       /* C = A + B                               */
  HS_OP_ADD_LN = 7,    /* Y = LayerNorm(A + B) * gamma + beta     */
  HS_OP_CONCAT = 8,    /* Y[:, i*c:(i+1)*c] = Z_i                 */
  HS_OP_ATTN_HEAD = 9, /* Z = softmax(s Q K^T) V W  (fused head)  */
  HS_OP_HEAD = 10,     /* [Q|K|V] = X Wqkv; Z = softmax(s Q K^T) V Wh (whole head) */
  HS_OP_COUNT = 11
} hs_op;

typedef enum {
  HS_MATH_TF32X3 = 0,   /* tcgen05 kind::tf32, 3-term split: fp32-accurate (default) */
  HS_MATH_TF32 = 1,     /* tcgen05 kind::tf32, single term (fast, ~1e-3)            */
  HS_MATH_FP32_SIMT = 2, /* CUDA-core fp32 FMA (diagnostic)                         */
  HS_MATH_BF16X3 = 3     /* GEMMs with resident (pre-split) B: kind::f16 with bf16 hi/lo
                            3-term split (~1e-5, 2x the tf32 MMA rate); other GEMMs
                            run TF32X3. B planes must be prepared with format 1. */
} hs_math;

#define HS_MAX_INPUTS 16
typedef struct {
  const void* in[HS_MAX_INPUTS]; /* input-side buffers in ascending arg position     */
  int64_t in_stride[HS_MAX_INPUTS]; /* per-instance stride in elements (0 = shared)  */
  int n_in;
  void* out;                        /* first output-side buffer                      */
  int64_t out_stride;               /* per-instance stride in elements               */
  int64_t dims[4];                  /* op-specific sizes             */
  float fparam[2];                  /* [0] scale s, [1] layer-norm eps               */
  const void* aux;                  /* GEMM: shared B pre-split by hs_gemm_split_weights, or NULL */
  /* Grouped GEMM launch (n_out > 1): n_out sibling GEMMs sharing A and dims
   * M, K, each with N = dims[1] columns; aux holds their planes concatenated
   * along N; member m writes outs[m] (per-instance stride out_strides[m]). */
  int n_out;
  void* outs[4];
  int64_t out_strides[4];
  /* GEMM output placement and epilogue (zero-initialised = plain C[M,N]):
   * out_ld  row stride of C in elements (0 = N): a GEMM can write one column
   *         block of a wider row-major matrix (e.g. its slot in a concat);
   * epilogue HS_EPI_SOFTMAX: C = row softmax(A·B · fparam[0]) over all N
   *         columns (N <= 128, tcgen05 math only) -- a GEMM fused with the
   *         softmax node that consumes it. */
  int64_t out_ld;
  int epilogue;
  /* HS_FLAG_* bits (0 = defaults). */
  int flags;
} hs_op_args;

#define HS_EPI_NONE 0
#define HS_EPI_SOFTMAX 1
/* No split-K: single-instance GEMMs otherwise add K-split partial sums with
 * red.global.add (fast for latency-bound launches, but the fp32 addition order
 * then varies from run to run). With this flag every launch is bit-reproducible. */
#define HS_FLAG_DETERMINISTIC 1
/* HS_OP_ATTN_HEAD ("attn_head"): in = {Q, K, V, W}, Q/K/V [S, dk] per instance,
 * W [dk, dw] shared and pre-split (aux, hs_gemm_split_weights_ex format 0);
 * dims = {S, dk, dw} with S <= 128, dk = dw = 64; fparam[0] = softmax scale;
 * out = Z [S, dw] (rows out_ld apart, 0 = dw). tcgen05 math (TF32X3 / TF32)
 * only. The transformer head of PAPER.md:323 as one node. */
/* HS_OP_HEAD (engine launch rewrite, no spec name): the head component of the
 * encoder DAG including its Q/K/V projections. in = {X, Wh planes}: X [S, D] per
 * instance, Wh [dk, dk] pre-split (format 0, stride 0); aux = Wq|Wk|Wv pre-split
 * side by side (hs_gemm_split_weights_strided, N = 3 dk, plane stride 3 dk D);
 * dims = {S, D, dk} with S <= 128, D % 32 == 0, dk = 64; fparam[0] = softmax
 * scale; out = Z [S, dk] (rows out_ld apart). TF32X3 / TF32 only. */

int hs_op_from_name(const char* name); /* -1 if unknown */
int hs_launch(hs_stream_t s, int op, const hs_op_args* args, int math_mode, int batch);
/* Resident-weight preparation for GEMM nodes: B ([K,N] if transposed == 0, else
 * [N,K]) -> K-major tf32 hi/lo planes `planes` = float[2][N][K]. Run once per
 * weight; pass `planes` as hs_op_args.aux on every launch that uses B. */
int hs_gemm_split_weights(hs_stream_t s, const void* B, int transposed, int64_t N, int64_t K, void* planes);
/* Same, writing hi at planes[n*K+k] and lo at planes[plane_stride + n*K+k] (elements):
 * used to lay several weights side by side for a grouped launch. */
int hs_gemm_split_weights_strided(hs_stream_t s, const void* B, int transposed, int64_t N, int64_t K, void* planes,
                                  int64_t plane_stride);
/* format 0 = tf32 hi/lo in fp32 containers (TF32X3/TF32), 1 = bf16 hi/lo (BF16X3). */
int hs_gemm_split_weights_ex(hs_stream_t s, const void* B, int transposed, int64_t N, int64_t K, void* planes,
                             int64_t plane_stride, int format);

int hs_host_callback(hs_stream_t s, void (*fn)(void*), void* user);
int hs_capture_begin(hs_stream_t s);
int hs_capture_end(hs_stream_t s, hs_graph_t* out);
int hs_graph_launch(hs_graph_t g, hs_stream_t s);
int hs_graph_destroy(hs_graph_t g);
/* Number of node-kernel launches issued through hs_launch so far (all threads). */
int64_t hs_launch_count(void);

/* ------------------------------------------------------ 3. engine */
typedef struct hs_engine* hs_engine_t;

/* config_json: {"spec": "<spec document>", "params": {..}, "gpu": 0,
 *   "policy": "clustering"|"eager"|"heft", "mode": "graph"|"dynamic",
 *   "batch": B, "slots": 2, "math": "tf32x3"|"tf32"|"simt",
 *   "cpu_devices": [..], "trace": false, "fuse": 3}
 * fuse (graph mode launch lowering): 0 one launch per ndrange,
 * 1 + grouped sibling GEMMs, 2 + chain rewrites, 3 (default) + whole-head launches.
 * Optional: "device_gpus": {"<logical device>": ordinal} (components across GPUs),
 * "domain_per_device": 0|1, "ramp": 1|0|R (first and last chunks of batch/4, off,
 * or R <= batch/2 instances when the bindings are host memory), "dynamic_fuse": 0|1 (dynamic mode issues the graph
 * plan's fused launches instead of one kernel per ndrange; InvalidParam when it
 * cannot apply: devices with different queue counts, or simt math),
 * "deterministic": 0|1 (HS_FLAG_DETERMINISTIC on every launch: no atomic split-K;
 * single-instance GEMMs use the cluster split-K with its in-order DSMEM reduction
 * either way, so this only excludes the red.add fallback),
 * "liveness": 1|0 (intermediate buffers share one arena per slot wherever the
 * DAG orders all their accesses; 0 = one allocation per output buffer),
 * "run_graph": 1|0 (graph mode on one GPU: a run of at most `batch` instances
 * replays one graph holding its copy-in, the plan and its copy-out, captured for
 * that (first, n) window; 0 = copies issued per run around the plan graph),
 * "zero_copy": 1|0 (with run_graph and n == batch: per-instance inputs / outputs
 * bound to dense, non-overlapping memory on this GPU are read / written in place
 * by the captured kernels instead of copied). */
int hs_engine_create(const char* config_json, hs_engine_t* out);
int hs_engine_destroy(hs_engine_t e);

/* Bind the isolated input (or isolated output) buffer (kernel, pos) to memory
 * holding `count` instances laid out `stride_bytes` apart (stride 0 = one copy
 * shared by every instance; such inputs are uploaded once and stay resident, and
 * `count` is ignored). on_device != 0 means `ptr` is device memory on the
 * engine's GPU. */
int hs_engine_bind(hs_engine_t e, int kernel, int pos, void* ptr, int64_t stride_bytes, int64_t count,
                   int on_device);

/* Execute `n_instances` DAG instances (instances [first, first+n) of the
 * bound arrays; InvalidParam unless 0 <= first and first + n <= count of every
 * per-instance binding). Blocks until done. elapsed_ns (optional) = device time
 * from the first to the last command, measured with CUDA events. */
int hs_engine_run(hs_engine_t e, int64_t first, int64_t n_instances, int64_t* elapsed_ns);

/* JSON introspection: what = "plan" | "stats" | "completions" | "trace". */
int hs_engine_info(hs_engine_t e, const char* what, char** out_json);

#ifdef __cplusplus
}
#endif

#endif /* HETSIM_C_H_ */
