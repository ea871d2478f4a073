// B200 executor: runs Alg. 1's dispatch(T, Q) on CUDA streams through the
// hs_* C ABI, and packages a DAG template + buffer bindings as an engine that
// executes a stream of instances (include/hetsim_c.h §3).
//
// Mapping:
//   queue i of a component on logical device d -> stream S[slot][d][i]
//   E_Q pair (a, b)                              -> record ev(a); S(b) waits ev(a)
//   inter edge (dependent read -> write)         -> record on the producer's read,
//                                                   consumer's write waits (data stays
//                                                   in HBM: the consumer aliases it)
//   callback mark                                -> cudaLaunchHostFunc (dynamic) /
//                                                   exclusivity join (graph)
//   ndrange                                      -> hs_launch (sm_100a kernels), one
//                                                   launch for all `batch` instances
//   isolated write/read                          -> H2D/D2H on the copy engines
#pragma once

#include <atomic>
#include <condition_variable>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <tuple>
#include <vector>

#include "hetsim/cq_builder.hpp"
#include "hetsim/scheduler.hpp"
#include "hetsim/spec_model.hpp"
#include "hetsim_c.h"

namespace hetsim {

struct EngineConfig {
  std::string spec_text;
  ParamMap params;
  int gpu = 0;
  Policy policy = Policy::clustering;
  bool graph_mode = true;
  int batch = 1;
  int slots = 2;
  int math = HS_MATH_TF32X3;
  std::set<int> cpu_devices;
  // Graph-mode launch lowering: 0 = one launch per ndrange, 1 = + grouped
  // sibling GEMMs, 2 = + chain rewrites (transpose folded into gemm_nt,
  // softmax as a GEMM epilogue, concat inputs written in place).
  int fuse = 3;
  // Record a timing-event pair around every command of the first batch of each
  // run (dynamic mode: as dispatched; graph mode: the plan issued directly).
  bool trace = false;
  // Components across GPUs: logical device -> physical GPU
  // ordinal (default: every logical device on `gpu`). Each distinct GPU is a
  // memory domain; an inter edge between domains is one peer copy on the
  // consumer's dependent write. domain_per_device makes every logical device its
  // own domain even on one GPU (exercises the peer path on a 1-GPU machine).
  std::map<int, int> device_gpus;
  bool domain_per_device = false;
  // Graph mode with host-memory inputs/outputs: first and last chunks of a run
  // use a second graph of ramp instances (shorter exposed copies): 1 = batch/4,
  // 0 = off, > 1 = that many instances (at most batch/2).
  int ramp = 1;
  // Dynamic mode with the graph plan's launch lowering (grouped / fused launches per
  // component); off by default: Alg. 1 as written launches one kernel per ndrange.
  bool dynamic_fuse = false;
  // HS_FLAG_DETERMINISTIC on every node launch (no split-K: bit-reproducible
  // single-instance GEMMs).
  bool deterministic = false;
  // Buffer-liveness planner: intermediates share one arena per slot when the DAG
  // orders all their accesses (false: one allocation per output buffer).
  bool liveness = true;
  // Graph mode, one memory domain: a run that is a single chunk (n <= batch, no ramp)
  // replays one graph holding its copy-in, the plan and its copy-out (captured per
  // (first, n) window), so a run costs one host submission.
  bool run_graph = true;
  // With run_graph and n == batch: device-resident per-instance inputs and outputs
  // (dense, on this GPU, not overlapping) are read and written in place by the
  // captured kernels instead of being copied into / out of the slot's buffers.
  bool zero_copy = true;
};

class Engine {
 public:
  explicit Engine(EngineConfig cfg);
  ~Engine();
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  // count = instances the memory holds (ignored when stride_bytes == 0)
  void bind(int kernel, int pos, void* ptr, int64_t stride_bytes, int64_t count, bool on_device);
  void run(int64_t first, int64_t n, int64_t* elapsed_ns);
  std::string info(const std::string& what) const;

  // Completion delivery from CUDA host callbacks (any thread).
  void push_completion(const Completion& c);
  // host callbacks: the per-callback record is created and consumed under mu_
  void* new_callback(const Completion& c);
  void deliver_callback(void* record);

  // Alg. 1 driven from outside (hetsim::CudaExecutor, include/hetsim/cuda_executor.hpp):
  // one scheduler run per ext_begin / ext_end over n <= batch instances, dynamic mode.
  void ext_begin(int64_t first, int64_t n);
  void ext_dispatch(const TaskComponent& t, const CommandQueueStructure& q);
  Completion ext_wait();
  int64_t ext_end();

 private:
  struct Node {
    int op = -1;
    std::vector<std::pair<int, int>> inputs;  // (kernel,pos) in arg order
    std::pair<int, int> output{-1, -1};
    int64_t dims[4] = {0, 0, 0, 0};
    float fparam[2] = {1.f, 1e-5f};
    // chain rewrites (graph mode, plan_fusion): the output lands at element
    // `out_off` of `output` with rows `out_ld` apart; `epilogue` is an
    // HS_EPI_* applied by the GEMM; an elided node has no launch of its own.
    int64_t out_off = 0, out_ld = 0;
    int epilogue = HS_EPI_NONE;
    float escale = 1.f;
    bool elided = false;
  };
  struct Binding {
    void* ptr = nullptr;
    int64_t stride = 0;  // bytes between instances; 0 = shared
    int64_t count = 0;   // instances held (per-instance bindings)
    bool on_device = false;
  };
  struct Group {  // one device allocation fed by one isolated binding (deduplicated)
    Binding b;
    int64_t bytes = 0;  // per instance
    bool resident = false;
    bool io = false;
  };
  struct Slot {
    std::map<std::pair<int, int>, void*> buf;  // (kernel,pos) -> device base for this slot
    std::map<std::pair<int, int>, void*> group_buf;  // per-instance groups: (group, domain) -> base
    hs_stream_t origin = nullptr;
    std::map<std::pair<int, int>, hs_stream_t> streams;  // (device, queue)
    std::map<std::pair<int, int>, hs_event_t> events;    // (component, event)
    std::map<int, std::pair<int, int>> edge_event;       // edge -> (component, event) of its dependent read
    std::map<int, hs_event_t> group_event;
    std::set<int> group_done;
    hs_graph_t graph = nullptr;
    hs_graph_t graph_small = nullptr;  // the plan at ramp_ instances
    // single-chunk runs (n <= batch): copy-in + plan + copy-out captured as one graph for
    // the run's instance window, so the host submits one launch per run
    hs_graph_t graph_run = nullptr;
    int64_t run_first = -1, run_n = -1;
    hs_event_t t_start = nullptr, t_end = nullptr;
    // several memory domains: per-domain copy streams joined to `origin`
    std::map<int, hs_stream_t> dorigin;
    std::map<int, hs_event_t> din, dout;
    hs_event_t copy_fork = nullptr;
    // one GPU, several per-instance input groups: copy-in streams forked from `origin`
    std::vector<hs_stream_t> copy_streams;
    std::vector<hs_event_t> copy_join;
  };

  void zero_copy_remap(Slot& sl, int64_t first, int64_t n);
  void build_nodes();
  void plan_buffers();
  std::map<std::pair<int, int>, std::set<int>> buffer_accessors() const;
  void place_slot_buffers();
  int64_t pooled_bytes_per_instance_ = 0, unpooled_bytes_per_instance_ = 0;
  void upload_resident();
  void capture(Slot& sl);
  void emit_plan(Slot& sl);
  void clear_trace();
  hs_stream_t stream(Slot& sl, int device, int queue);
  hs_event_t event(Slot& sl, int comp, int ev, int dom = -1);
  void issue(Slot& sl, const TaskComponent& t, const CommandQueueStructure& q, int prev_comp,
             const CommandQueueStructure* prev_q, bool graph, int64_t first, int64_t n);
  void launch_node(Slot& sl, hs_stream_t s, int kernel);
  void copy_in(Slot& sl, hs_stream_t s, int group, int64_t first, int64_t n, int dom);
  void copy_out(Slot& sl, hs_stream_t s, int64_t first, int64_t n, int dom);
  void copies(Slot& sl, int64_t first, int64_t n, bool in);
  void place_components();
  int kdom(int kernel) const;
  void* dalloc(int dom, int64_t bytes);
  hs_stream_t dstream(Slot& sl, int dom);
  void run_dynamic(Slot& sl, int64_t first, int64_t n);
  void check_range(int64_t first, int64_t n) const;
  void plan_once();
  void reset_dynamic_state(Slot& sl);
  void join_dynamic_streams(Slot& sl);
  int64_t ext_first_ = 0, ext_n_ = 0;
  bool ext_open_ = false;
  Completion wait_completion();


  EngineConfig cfg_;
  DagSpec g_;
  Platform platform_;
  std::unique_ptr<Scheduler> sched_;
  ScheduleResult plan_;
  std::map<int, Node> nodes_;
  std::map<std::pair<int, int>, Binding> bindings_;
  std::vector<Group> groups_;
  std::map<std::pair<int, int>, int> group_of_;                 // isolated input (kernel,pos) -> group
  std::map<std::pair<int, int>, std::pair<int, int>> alias_;    // input (kernel,pos) -> producer (kernel,pos)
  std::map<std::pair<int, int>, std::pair<int, int>> io_copy_;  // io input fed by an edge -> producer
  std::map<std::pair<int, int>, int64_t> bytes_;                // (kernel,pos) -> bytes per instance
  std::vector<std::pair<int, int>> outputs_;                    // isolated outputs with a binding
  // zero-copy capture of a whole-run graph: groups / outputs read or written in place
  std::set<int> skip_groups_;
  std::set<std::pair<int, int>> skip_outputs_;
  int64_t zero_copy_groups_ = 0, zero_copy_outputs_ = 0;
  std::map<std::pair<int, int>, void*> resident_;  // (resident group, domain) -> device copy
  // resident GEMM weights pre-split into tf32 hi/lo planes: (group, transposed) -> planes
  struct Planes {
    void* ptr = nullptr;
    int gi = -1;
    bool nt = false;
    int64_t n = 0, k = 0;
    int dom = 0;
  };
  std::map<std::tuple<int, bool, int>, Planes> planes_;  // (group, transposed, domain)
  std::map<int, void*> node_planes_;  // kernel -> planes
  std::map<int, void*> head_qkv_planes_;  // HS_OP_HEAD kernel -> its absorbed group's Wq|Wk|Wv planes
  std::map<std::pair<int, int>, Planes> attn_planes_;  // (resident group, domain) -> tf32 planes for fused heads

  // Grouped launches (graph mode): sibling GEMM ndranges of one component that
  // share their A input, have resident B and no intra-component producer run as
  // one tcgen05 launch with their B planes side by side (N = members x 64).
  struct FuseGroup {
    int component = -1;
    std::vector<int> kernels;  // members, ascending ndrange event
    std::vector<int> events;
    void* planes = nullptr;
    int64_t n = 0, k = 0;  // per member
    bool absorbed = false;  // computed inside a whole-head launch (head_fused rule): no launch of its own
  };
  void plan_fusion();
  void plan_chain_rewrites();
  std::map<std::string, int64_t> rewrites_;  // rule -> times applied
  // weight planes: bf16 hi/lo for BF16X3, tf32 hi/lo (fp32 containers) otherwise
  int plane_format() const { return cfg_.math == HS_MATH_BF16X3 ? 1 : 0; }
  int64_t plane_elem_bytes() const { return cfg_.math == HS_MATH_BF16X3 ? 2 : 4; }
  std::vector<FuseGroup> fuse_groups_;
  std::map<std::pair<int, int>, int> fuse_leader_;  // (component, ndrange event) -> group
  std::map<std::pair<int, int>, int> fuse_member_;  // (component, ndrange event) -> group (non-leaders)
  hs_ctx_t ctx_ = nullptr;  // domain 0
  std::vector<hs_ctx_t> dctx_;       // memory domain -> context
  std::vector<int> dom_gpu_;         // memory domain -> GPU ordinal
  std::map<int, int> dev_dom_;       // logical device -> domain
  std::map<int, int> comp_dom_;      // component -> domain (graph mode plan)
  std::map<int, int> kernel_dom_;    // kernel -> domain
  std::map<hs_stream_t, int> stream_dom_;
  std::map<std::pair<int, int>, std::pair<int, int>> peer_in_;  // input fed across domains -> producer
  bool capture_ok_ = true;           // one physical GPU: the plan is captured into graphs
  int64_t ramp_ = 0;                 // small-graph batch (0: no ramp)
  bool dyn_fused_ = false;           // dynamic mode issues the fused launches
  int64_t cur_batch_ = 0;            // instances of the plan being emitted (0: cfg_.batch)
  int64_t nb() const { return cur_batch_ ? cur_batch_ : cfg_.batch; }
  std::vector<Slot> slots_;
  bool planned_ = false;
  bool resident_uploaded_ = false;
  int64_t device_bytes_ = 0;
  int64_t launches_per_batch_ = 0;
  int64_t runs_ = 0, batches_run_ = 0;
  std::vector<std::pair<int, void*>> allocations_;  // (domain, pointer)

  // dynamic-mode completion queue (MPSC: CUDA callback threads -> scheduler thread)
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<Completion> done_q_;
  std::atomic<int> pending_{0};
  static constexpr int kSpinUs = 2000;
  int64_t host_dispatch_ns_ = 0, host_wait_ns_ = 0, host_dispatches_ = 0;
  std::vector<Completion> last_log_;
  struct TraceRec {
    int component = -1, event = -1, kind = 0, kernel = -1, device = -1, queue = -1;
    std::string label;
    hs_event_t t0 = nullptr, t1 = nullptr;
  };
  bool tracing_ = false;
  std::vector<TraceRec> trace_;
  std::vector<DispatchRecord> trace_dispatch_;
  std::vector<DispatchRecord> last_dispatches_;
};

}  // namespace hetsim
