// B200 executor / engine. See engine.hpp for the command -> CUDA mapping.
//
// Two execution modes over the same issue() path:
//  * dynamic — Alg. 1 literally: the Scheduler calls CudaDispatch::dispatch
//    for every (T, d) it selects; completions of callback-marked commands
//    come back through cudaLaunchHostFunc -> MPSC queue -> Scheduler::cb.
//    A logical device stays locked until its component's terminal commands
//    complete.
//  * graph   — the same Scheduler is run once against PlanExecutor to fix the
//    dispatch sequence; issue() then records that sequence into a CUDA graph
//    per instance slot (stream capture over the per-queue streams). Device
//    exclusivity becomes an event join on the previous component's terminal
//    commands, so no host round trip sits between components. Steady-state
//    batches are copy-in -> graph launch -> copy-out on the slot's origin
//    stream, slots alternating so that copies overlap compute.
#include "engine.hpp"

#include <algorithm>
#include <chrono>
#include <cstring>
#include <tuple>

#include "../core/json.hpp"
#include "hetsim/errors.hpp"

extern "C" int hs__set_error(int status, int errc, const char* msg);

namespace hetsim {

namespace {

void hs_ok(int r, const char* what) {
  if (r == HS_OK) return;
  const int errc = hs_last_errc();
  std::string msg = std::string(what) + ": " + hs_last_error();
  fail(errc == static_cast<int>(Errc::invalid_param) ? Errc::invalid_param : Errc::device_error, msg);
}

struct CbData {
  Engine* engine;
  Completion c;
};

// Runs on a CUDA driver thread. The record was written under the engine's mutex
// before the callback was enqueued and is read under it here: the mutex, not the
// driver's internal hand-off, orders the two accesses (what ThreadSanitizer checks,
// `make tsan`).
void CUDART_CB_trampoline(void* p) {
  auto* d = static_cast<CbData*>(p);
  d->engine->deliver_callback(d);
}

std::vector<long long> var_values(const KernelSpec& k, const ParamMap& params) {
  std::vector<const VarArg*> vs;
  for (const auto& v : k.var_args) vs.push_back(&v);
  std::sort(vs.begin(), vs.end(), [](const VarArg* a, const VarArg* b) { return a->pos < b->pos; });
  std::vector<long long> out;
  for (const VarArg* v : vs) out.push_back(eval_expr(v->value, params));
  return out;
}

}  // namespace

// Executor used in dynamic mode: Alg. 1 dispatch -> Engine::issue (the same
// path a caller-driven hetsim::CudaExecutor takes through ext_dispatch).
class CudaDispatch : public Executor {
 public:
  explicit CudaDispatch(Engine& e) : e_(e) {}
  void dispatch(const TaskComponent& t, const CommandQueueStructure& q) override { e_.ext_dispatch(t, q); }
  Completion wait_next() override { return e_.ext_wait(); }

 private:
  Engine& e_;
};

Engine::Engine(EngineConfig cfg) : cfg_(std::move(cfg)) {
  if (cfg_.batch < 1) fail(Errc::invalid_param, "batch must be >= 1");
  if (cfg_.slots < 1) cfg_.slots = 1;
  g_ = parse_spec(cfg_.spec_text, cfg_.params);
  platform_ = Platform::from_spec(g_, cfg_.cpu_devices, 1);
  for (const auto& d : platform_.devices)
    if (d.type == DeviceType::cpu)
      fail(Errc::invalid_param, "device " + std::to_string(d.id) + " is a CPU device; the B200 executor has no CPU path");
  sched_ = std::make_unique<Scheduler>(g_, platform_, Profiles{}, cfg_.policy);
  build_nodes();
  // Memory domains: one per physical GPU the logical devices map to (or per
  // logical device with domain_per_device). Domain 0 hosts the origin streams.
  std::map<long long, int> dom_of_key;
  for (const auto& d : platform_.devices) {
    auto it = cfg_.device_gpus.find(d.id);
    const int gpu = it == cfg_.device_gpus.end() ? cfg_.gpu : it->second;
    const long long key = cfg_.domain_per_device ? (1LL << 40) + d.id : gpu;
    auto [pos, fresh] = dom_of_key.emplace(key, int(dom_gpu_.size()));
    if (fresh) dom_gpu_.push_back(gpu);
    dev_dom_[d.id] = pos->second;
  }
  if (dom_gpu_.empty()) dom_gpu_.push_back(cfg_.gpu);
  if (dom_gpu_.size() > 1 && !cfg_.graph_mode)
    fail(Errc::invalid_param, "components mapped to several GPUs need graph mode (the plan fixes their placement)");
  for (int gpu : dom_gpu_) {
    hs_ctx_t c = nullptr;
    hs_ok(hs_ctx_create(gpu, &c), "hs_ctx_create");
    dctx_.push_back(c);
  }
  ctx_ = dctx_.front();
  for (size_t a = 0; a < dctx_.size(); ++a)
    for (size_t b = 0; b < dctx_.size(); ++b)
      if (dom_gpu_[a] != dom_gpu_[b]) {
        hs_ok(hs_ctx_enable_peer(dctx_[a], dctx_[b]), "hs_ctx_enable_peer");
        capture_ok_ = false;  // the plan is issued directly on several GPUs
      }
}

int Engine::kdom(int kernel) const {
  auto it = kernel_dom_.find(kernel);
  return it == kernel_dom_.end() ? 0 : it->second;
}

void* Engine::dalloc(int dom, int64_t bytes) {
  void* p = nullptr;
  hs_ok(hs_malloc(dctx_[size_t(dom)], size_t(bytes), &p), "hs_malloc");
  allocations_.push_back({dom, p});
  device_bytes_ += bytes;
  return p;
}

hs_stream_t Engine::dstream(Slot& sl, int dom) {
  if (dom == 0) return sl.origin;
  auto it = sl.dorigin.find(dom);
  if (it != sl.dorigin.end()) return it->second;
  hs_stream_t s = nullptr;
  hs_ok(hs_stream_create(dctx_[size_t(dom)], 0, &s), "hs_stream_create");
  stream_dom_[s] = dom;
  hs_event_t a = nullptr, b = nullptr;
  hs_ok(hs_event_create(dctx_[size_t(dom)], 0, &a), "hs_event_create");
  hs_ok(hs_event_create(dctx_[size_t(dom)], 0, &b), "hs_event_create");
  sl.din[dom] = a;
  sl.dout[dom] = b;
  sl.dorigin[dom] = s;
  return s;
}

// Graph mode: the plan's component -> logical device choice fixes every
// kernel's memory domain before buffers are placed.
void Engine::place_components() {
  for (const auto& rec : plan_.dispatches) comp_dom_[rec.component] = dev_dom_.at(rec.device);
  for (const auto& t : sched_->components())
    for (int k : t.kernel_ids) kernel_dom_[k] = comp_dom_.count(t.id) ? comp_dom_.at(t.id) : 0;
}

Engine::~Engine() {
  if (!ctx_) return;
  for (hs_ctx_t c : dctx_) hs_ctx_sync(c);
  { std::lock_guard<std::mutex> lk(mu_); }  // every host callback has left deliver_callback
  clear_trace();
  for (auto& sl : slots_) {
    hs_graph_destroy(sl.graph);
    hs_graph_destroy(sl.graph_small);
    hs_graph_destroy(sl.graph_run);
    for (auto& [k, e] : sl.events) hs_event_destroy(e);
    for (auto& [k, e] : sl.group_event) hs_event_destroy(e);
    for (auto& [k, e] : sl.din) hs_event_destroy(e);
    for (auto& [k, e] : sl.dout) hs_event_destroy(e);
    hs_event_destroy(sl.copy_fork);
    for (hs_event_t e : sl.copy_join) hs_event_destroy(e);
    for (hs_stream_t cs : sl.copy_streams) hs_stream_destroy(cs);
    hs_event_destroy(sl.t_start);
    hs_event_destroy(sl.t_end);
    for (auto& [k, s] : sl.streams) hs_stream_destroy(s);
    for (auto& [k, s] : sl.dorigin) hs_stream_destroy(s);
    hs_stream_destroy(sl.origin);
  }
  for (auto [dom, p] : allocations_) hs_free(dctx_[size_t(dom)], p);
  for (hs_ctx_t c : dctx_) hs_ctx_destroy(c);
}

void Engine::build_nodes() {
  for (const auto& k : g_.kernels) {
    Node nd;
    nd.op = hs_op_from_name(k.name.c_str());
    if (nd.op < 0) fail(Errc::invalid_param, "kernel " + std::to_string(k.id) + ": no sm_100a operator '" + k.name + "'");
    for (const auto* b : k.input_side()) nd.inputs.push_back({k.id, b->pos});
    auto outs = k.output_side();
    if (outs.empty()) fail(Errc::invalid_param, "kernel " + std::to_string(k.id) + " has no output buffer");
    nd.output = {k.id, outs.front()->pos};
    for (const auto* list : {&k.input_buffers, &k.output_buffers, &k.io_buffers})
      for (const auto& b : *list) {
        if (b.type != ElemType::f32)
          fail(Errc::invalid_param, "kernel " + std::to_string(k.id) + ": only float32 buffers are supported");
        bytes_[{k.id, b.pos}] = buffer_bytes(b, g_.params);
      }
    auto v = var_values(k, g_.params);
    auto elems = [&](std::pair<int, int> key) { return bytes_.at(key) / 4; };
    auto need = [&](bool ok, const char* what) {
      if (!ok) fail(Errc::invalid_param, "kernel " + std::to_string(k.id) + " (" + k.name + "): " + what);
    };
    const size_t nin = nd.inputs.size();
    switch (nd.op) {
      case HS_OP_GEMM:
      case HS_OP_GEMM_NT:
      case HS_OP_GEMM_RELU:
        need(v.size() >= 3 && nin == 2, "expects (A, B, C, M, N, K)");
        for (int i = 0; i < 3; ++i) nd.dims[i] = v[size_t(i)];
        need(elems(nd.inputs[0]) == v[0] * v[2], "A size != M*K");
        need(elems(nd.inputs[1]) == v[1] * v[2], "B size != K*N");
        need(elems(nd.output) == v[0] * v[1], "C size != M*N");
        break;
      case HS_OP_TRANSPOSE:
        need(v.size() >= 2 && nin == 1, "expects (A, B, R, C)");
        nd.dims[0] = v[0];
        nd.dims[1] = v[1];
        need(elems(nd.inputs[0]) == v[0] * v[1] && elems(nd.output) == v[0] * v[1], "size != R*C");
        break;
      case HS_OP_SCALE:
        need(v.size() >= 3 && nin == 1 && v[2] != 0, "expects (A, B, n, num, den)");
        nd.dims[0] = v[0];
        nd.fparam[0] = float(double(v[1]) / double(v[2]));
        need(elems(nd.inputs[0]) == v[0] && elems(nd.output) == v[0], "size != n");
        break;
      case HS_OP_SOFTMAX:
        need(v.size() >= 2 && nin == 1, "expects (A, B, rows, cols[, num, den])");
        nd.dims[0] = v[0];
        nd.dims[1] = v[1];
        nd.fparam[0] = v.size() >= 4 && v[3] != 0 ? float(double(v[2]) / double(v[3])) : 1.f;
        need(elems(nd.inputs[0]) == v[0] * v[1] && elems(nd.output) == v[0] * v[1], "size != rows*cols");
        need(v[1] <= 1024, "cols > 1024");
        break;
      case HS_OP_ADD:
        need(v.size() >= 1 && nin == 2, "expects (A, B, C, n)");
        nd.dims[0] = v[0];
        need(elems(nd.inputs[0]) == v[0] && elems(nd.inputs[1]) == v[0] && elems(nd.output) == v[0], "size != n");
        break;
      case HS_OP_ADD_LN:
        need(v.size() >= 2 && nin == 4, "expects (A, B, gamma, beta, Y, rows, cols)");
        nd.dims[0] = v[0];
        nd.dims[1] = v[1];
        need(elems(nd.inputs[0]) == v[0] * v[1] && elems(nd.inputs[1]) == v[0] * v[1] &&
                 elems(nd.output) == v[0] * v[1],
             "size != rows*cols");
        need(elems(nd.inputs[2]) == v[1] && elems(nd.inputs[3]) == v[1], "gamma/beta size != cols");
        need(v[1] <= 1024, "cols > 1024");
        break;
      case HS_OP_CONCAT:
        need(v.size() >= 2 && nin >= 1 && nin <= HS_MAX_INPUTS, "expects (Z0..Zn-1, Y, rows, cols_each)");
        nd.dims[0] = v[0];
        nd.dims[1] = v[1];
        for (auto in : nd.inputs) need(elems(in) == v[0] * v[1], "input size != rows*cols_each");
        need(elems(nd.output) == v[0] * v[1] * int64_t(nin), "output size != rows*cols_each*count");
        break;
      case HS_OP_ATTN_HEAD:
        need(v.size() >= 3 && nin == 4, "expects (Q, K, V, W, Z, S, dk, dw[, num, den])");
        for (int i = 0; i < 3; ++i) nd.dims[i] = v[size_t(i)];
        nd.fparam[0] = v.size() >= 5 && v[4] != 0 ? float(double(v[3]) / double(v[4])) : 1.f;
        for (size_t i = 0; i < 3; ++i) need(elems(nd.inputs[i]) == v[0] * v[1], "Q/K/V size != S*dk");
        need(elems(nd.inputs[3]) == v[1] * v[2], "W size != dk*dw");
        need(elems(nd.output) == v[0] * v[2], "Z size != S*dw");
        break;
      default: break;
    }
    nodes_[k.id] = nd;
  }
}

void Engine::bind(int kernel, int pos, void* ptr, int64_t stride_bytes, int64_t count, bool on_device) {
  if (planned_) fail(Errc::invalid_param, "bindings are frozen after the first run");
  const BufferSpec* b = g_.kernel(kernel).buffer_at(pos);
  if (!b) fail(Errc::invalid_param, "kernel " + std::to_string(kernel) + " has no buffer at position " + std::to_string(pos));
  if (!ptr) fail(Errc::invalid_param, "null binding");
  if (stride_bytes < 0) fail(Errc::invalid_param, "negative stride");
  if (stride_bytes > 0 && count < 1) fail(Errc::invalid_param, "a per-instance binding needs count >= 1");
  bindings_[{kernel, pos}] = Binding{ptr, stride_bytes, stride_bytes > 0 ? count : 0, on_device};
}

void Engine::plan_buffers() {
  auto producers = g_.producer_edge();
  auto ec = sched_->edge_classes();
  std::map<std::tuple<void*, int64_t, int64_t, bool>, int> dedupe;
  for (const auto& k : g_.kernels) {
    for (const auto* b : k.input_side()) {
      std::pair<int, int> key{k.id, b->pos};
      auto pe = producers.find(key);
      if (pe != producers.end()) {
        const DagEdge& e = g_.edges[size_t(pe->second)];
        const std::pair<int, int> src{e.src_kernel, e.src_pos};
        if (kdom(k.id) != kdom(e.src_kernel)) peer_in_[key] = src;  // one peer copy per batch
        else if (b->kind == BufferKind::io) io_copy_[key] = src;
        else alias_[key] = src;
        continue;
      }
      auto bi = bindings_.find(key);
      if (bi == bindings_.end())
        fail(Errc::invalid_param, "isolated input (" + std::to_string(k.id) + "," + std::to_string(b->pos) + ") is not bound");
      Group gr;
      gr.b = bi->second;
      gr.bytes = bytes_.at(key);
      gr.resident = gr.b.stride == 0;
      gr.io = b->kind == BufferKind::io;
      if (gr.io && gr.resident) fail(Errc::invalid_param, "an io buffer cannot be bound as shared (stride 0)");
      if (!gr.io) {
        auto dk = std::make_tuple(gr.b.ptr, gr.b.stride, gr.bytes, gr.b.on_device);
        auto it = dedupe.find(dk);
        if (it != dedupe.end()) {
          group_of_[key] = it->second;
          continue;
        }
        dedupe[dk] = int(groups_.size());
      }
      group_of_[key] = int(groups_.size());
      groups_.push_back(gr);
    }
    for (const auto* b : k.output_side()) {
      std::pair<int, int> key{k.id, b->pos};
      if (ec.read_class.at(key) == CopyClass::isolated && bindings_.count(key)) outputs_.push_back(key);
    }
  }
  // resident groups: one copy per domain that reads them
  for (const auto& [key, gi] : group_of_)
    if (groups_[size_t(gi)].resident && !resident_.count({gi, kdom(key.first)}))
      resident_[{gi, kdom(key.first)}] = dalloc(kdom(key.first), groups_[size_t(gi)].bytes);
  // GEMM nodes whose B operand is a resident weight get it pre-split once
  // (tf32 hi/lo, K-major) so the tensor cores are fed by TMA with no conversion.
  if (cfg_.math != HS_MATH_FP32_SIMT) {
    for (const auto& [kid, nd] : nodes_) {
      const int dom = kdom(kid);
      if (nd.op == HS_OP_ATTN_HEAD) {  // spec-level fused head: W must be resident, tf32 planes
        auto gi = group_of_.find(nd.inputs[3]);
        if (gi == group_of_.end() || !groups_[size_t(gi->second)].resident)
          fail(Errc::invalid_param, "attn_head kernel " + std::to_string(kid) + ": W must be bound as shared (resident)");
        auto it = attn_planes_.find({gi->second, dom});
        if (it == attn_planes_.end()) {
          Planes pl;
          pl.gi = gi->second;
          pl.n = nd.dims[2];
          pl.k = nd.dims[1];
          pl.dom = dom;
          pl.ptr = dalloc(dom, 2 * pl.n * pl.k * 4);
          it = attn_planes_.emplace(std::make_pair(gi->second, dom), pl).first;
        }
        node_planes_[kid] = it->second.ptr;
        continue;
      }
      if (nd.op != HS_OP_GEMM && nd.op != HS_OP_GEMM_NT && nd.op != HS_OP_GEMM_RELU) continue;
      auto gi = group_of_.find(nd.inputs[1]);
      if (gi == group_of_.end() || !groups_[size_t(gi->second)].resident) continue;
      const bool nt = nd.op == HS_OP_GEMM_NT;
      auto key = std::make_tuple(gi->second, nt, dom);
      auto it = planes_.find(key);
      if (it == planes_.end()) {
        Planes pl;
        pl.gi = gi->second;
        pl.nt = nt;
        pl.n = nd.dims[1];
        pl.k = nd.dims[2];
        pl.dom = dom;
        pl.ptr = dalloc(dom, 2 * pl.n * pl.k * plane_elem_bytes());
        it = planes_.emplace(key, pl).first;
      }
      node_planes_[kid] = it->second.ptr;
    }
  }
  launches_per_batch_ = int64_t(g_.kernels.size());
}

// Which launch of the plan touches which buffer, after the launch rewrites.
// Returns, for every output-side buffer (kernel,pos), the kernels whose
// launches (or dependent-write copies) read or write it. An accessor stands for
// the position of that kernel's ndrange in the plan; a grouped launch counts as
// every member (it starts after all members' inputs are ready, and every
// member's event completes after it). Buffers no launch touches (outputs of
// elided nodes, absorbed intermediates) get no entry.
std::map<std::pair<int, int>, std::set<int>> Engine::buffer_accessors() const {
  std::map<std::pair<int, int>, std::set<int>> acc;
  auto phys = [&](std::pair<int, int> key) {
    auto al = alias_.find(key);
    return al == alias_.end() ? key : al->second;
  };
  const bool fused = cfg_.graph_mode || dyn_fused_;
  std::set<int> grouped_members;
  if (fused)
    for (const auto& fg : fuse_groups_) {
      grouped_members.insert(fg.kernels.begin(), fg.kernels.end());
      if (fg.absorbed) continue;
      const Node& lead = nodes_.at(fg.kernels[0]);
      for (int m : fg.kernels) {
        acc[phys(lead.inputs[0])].insert(fg.kernels.begin(), fg.kernels.end());
        acc[nodes_.at(m).output].insert(fg.kernels.begin(), fg.kernels.end());
      }
    }
  for (const auto& [kid, nd] : nodes_) {
    if (grouped_members.count(kid) || nd.elided) continue;
    for (const auto& in : nd.inputs) {
      acc[phys(in)].insert(kid);
      auto io = io_copy_.find(in);
      if (io != io_copy_.end()) acc[io->second].insert(kid);
    }
    acc[nd.output].insert(kid);
  }
  // dependent-write copies (io inputs, peer copies) run on the consumer's queue
  for (const auto& [key, src] : io_copy_) {
    acc[key].insert(key.first);
    acc[src].insert(key.first);
  }
  for (const auto& [key, src] : peer_in_) acc[src].insert(key.first);
  return acc;
}

// Per-slot device memory with buffer liveness (graph and dynamic mode alike).
// Fixed allocations: per-instance input groups (written by copy-in before the
// plan), bound isolated outputs (read by copy-out after it), io buffers and
// peer-copy targets. Every other output buffer lives in one arena per (slot,
// memory domain), at an offset chosen first-fit in plan order: two buffers may
// share bytes only when every launch touching one is a proper DAG ancestor of
// every launch touching the other. DAG edges are exactly what the plan
// enforces (same-queue order, E_Q events, inter-edge events), so the earlier
// buffer's last access completes before the later buffer's first write, in any
// interleaving of the streams.
void Engine::place_slot_buffers() {
  const int64_t B = cfg_.batch;
  const auto acc = buffer_accessors();
  // proper-ancestor bitsets over kernel indices
  const size_t K = g_.kernels.size(), W = (K + 63) / 64;
  std::vector<std::vector<uint64_t>> anc(K, std::vector<uint64_t>(W, 0));
  std::map<int, int> topo_pos;
  {
    const auto order = g_.topo_order();
    for (size_t i = 0; i < order.size(); ++i) topo_pos[order[i]] = int(i);
    const auto preds = g_.kernel_predecessors();
    for (int v : order) {
      auto& av = anc[size_t(g_.index_of(v))];
      auto pit = preds.find(v);
      if (pit == preds.end()) continue;
      for (int u : pit->second) {
        const size_t ui = size_t(g_.index_of(u));
        av[ui / 64] |= uint64_t(1) << (ui % 64);
        for (size_t w = 0; w < W; ++w) av[w] |= anc[ui][w];
      }
    }
  }
  auto before = [&](const std::set<int>& a, const std::set<int>& b) {  // every a strictly precedes every b
    for (int y : b) {
      const auto& ay = anc[size_t(g_.index_of(y))];
      for (int x : a) {
        const size_t xi = size_t(g_.index_of(x));
        if (!(ay[xi / 64] >> (xi % 64) & 1)) return false;
      }
    }
    return true;
  };
  std::set<std::pair<int, int>> fixed(outputs_.begin(), outputs_.end());
  for (const auto& k : g_.kernels)
    for (const auto* b : k.output_side())
      if (b->kind == BufferKind::io) fixed.insert({k.id, b->pos});
  for (const auto& [key, gi] : group_of_) fixed.insert(key);
  for (const auto& [key, src] : peer_in_) fixed.insert(key);
  struct Placed {
    std::pair<int, int> key;
    const std::set<int>* acc;
    int64_t off, size;  // per-instance units
    int dom;
  };
  std::vector<Placed> pooled;
  for (const auto& k : g_.kernels)
    for (const auto* b : k.output_side()) {
      const std::pair<int, int> key{k.id, b->pos};
      auto it = acc.find(key);
      if (!cfg_.liveness) fixed.insert(key);  // one allocation per output buffer
      if (fixed.count(key) || it == acc.end()) continue;
      pooled.push_back({key, &it->second, 0, (bytes_.at(key) + 127) / 128 * 128, kdom(k.id)});
    }
  auto first_pos = [&](const Placed& p) {
    int m = 1 << 30;
    for (int x : *p.acc) m = std::min(m, topo_pos.at(x));
    return m;
  };
  std::stable_sort(pooled.begin(), pooled.end(),
                   [&](const Placed& a, const Placed& b) { return first_pos(a) < first_pos(b); });
  std::map<int, int64_t> arena;  // domain -> per-instance units
  for (size_t i = 0; i < pooled.size(); ++i) {
    Placed& p = pooled[i];
    std::vector<std::pair<int64_t, int64_t>> busy;
    for (size_t j = 0; j < i; ++j) {
      const Placed& q = pooled[j];
      if (q.dom == p.dom && !before(*q.acc, *p.acc) && !before(*p.acc, *q.acc)) busy.push_back({q.off, q.off + q.size});
    }
    std::sort(busy.begin(), busy.end());
    int64_t off = 0;
    for (auto [lo, hi] : busy) {
      if (off + p.size <= lo) break;
      off = std::max(off, hi);
    }
    p.off = off;
    arena[p.dom] = std::max(arena[p.dom], off + p.size);
  }
  int64_t unpooled = 0;
  for (const auto& k : g_.kernels)
    for (const auto* b : k.output_side()) unpooled += bytes_.at({k.id, b->pos});
  pooled_bytes_per_instance_ = 0;
  for (const auto& [d, units] : arena) pooled_bytes_per_instance_ += units;
  unpooled_bytes_per_instance_ = unpooled;
  slots_.resize(size_t(cfg_.slots));
  for (auto& sl : slots_) {
    std::map<int, char*> base;
    for (const auto& [d, units] : arena) base[d] = static_cast<char*>(dalloc(d, units * B));
    for (const auto& p : pooled) sl.buf[p.key] = base.at(p.dom) + p.off * B;
    for (const auto& k : g_.kernels)
      for (const auto* b : k.output_side()) {
        const std::pair<int, int> key{k.id, b->pos};
        if (fixed.count(key)) sl.buf[key] = dalloc(kdom(k.id), bytes_.at(key) * B);
      }
    for (const auto& [key, gi] : group_of_) {
      const Group& gr = groups_[size_t(gi)];
      const int dom = kdom(key.first);
      if (gr.resident) {
        sl.buf[key] = resident_.at({gi, dom});
        continue;
      }
      if (gr.io) sl.group_buf[{gi, dom}] = sl.buf.at(key);  // io group lives in the (kernel,pos) allocation
      else if (!sl.group_buf.count({gi, dom})) sl.group_buf[{gi, dom}] = dalloc(dom, gr.bytes * B);
      sl.buf[key] = sl.group_buf.at({gi, dom});
    }
    for (const auto& [key, src] : alias_) {
      auto it = sl.buf.find(src);
      if (it != sl.buf.end()) sl.buf[key] = it->second;  // (no entry: read by no launch)
    }
    for (const auto& [key, src] : peer_in_)
      if (!sl.buf.count(key)) sl.buf[key] = dalloc(kdom(key.first), bytes_.at(key) * B);  // io inputs reuse their output
    hs_ok(hs_stream_create(ctx_, 0, &sl.origin), "hs_stream_create");
    stream_dom_[sl.origin] = 0;
    hs_ok(hs_event_create(ctx_, 1, &sl.t_start), "hs_event_create");
    hs_ok(hs_event_create(ctx_, 1, &sl.t_end), "hs_event_create");
    if (dctx_.size() > 1) {
      hs_ok(hs_event_create(ctx_, 0, &sl.copy_fork), "hs_event_create");
      for (size_t d = 1; d < dctx_.size(); ++d) dstream(sl, int(d));
    }
  }
}

void Engine::upload_resident() {
  if (resident_uploaded_) return;
  Slot& s0 = slots_.front();
  for (const auto& [gd, dst] : resident_) {
    const Group& gr = groups_[size_t(gd.first)];
    hs_ok(hs_memcpy_2d(dstream(s0, gd.second), dst, size_t(gr.bytes), gr.b.ptr, size_t(gr.bytes), size_t(gr.bytes), 1,
                       gr.b.on_device ? 2 : 0),
          "resident upload");
  }
  for (const auto& [key, pl] : planes_)
    hs_ok(hs_gemm_split_weights_ex(dstream(s0, pl.dom), resident_.at({pl.gi, pl.dom}), pl.nt ? 1 : 0, pl.n, pl.k,
                                   pl.ptr, pl.n * pl.k, plane_format()),
          "split weights");
  for (const auto& [key, pl] : attn_planes_)
    hs_ok(hs_gemm_split_weights_ex(dstream(s0, pl.dom), resident_.at({pl.gi, pl.dom}), 0, pl.n, pl.k, pl.ptr,
                                   pl.n * pl.k, 0),
          "split attention weights");
  for (const auto& fg : fuse_groups_) {
    const int64_t members = int64_t(fg.kernels.size());
    const int dom = comp_dom_.count(fg.component) ? comp_dom_.at(fg.component) : 0;
    for (int64_t m = 0; m < members; ++m) {
      const int gi = group_of_.at(nodes_.at(fg.kernels[size_t(m)]).inputs[1]);
      hs_ok(hs_gemm_split_weights_ex(dstream(s0, dom), resident_.at({gi, dom}), 0, fg.n, fg.k,
                                     static_cast<char*>(fg.planes) + m * fg.n * fg.k * plane_elem_bytes(),
                                     members * fg.n * fg.k, plane_format()),
            "split grouped weights");
    }
  }
  hs_ok(hs_stream_sync(s0.origin), "resident upload sync");
  for (auto& [d, st] : s0.dorigin) hs_ok(hs_stream_sync(st), "resident upload sync");
  resident_uploaded_ = true;
}

hs_stream_t Engine::stream(Slot& sl, int device, int queue) {
  auto key = std::make_pair(device, queue);
  auto it = sl.streams.find(key);
  if (it != sl.streams.end()) return it->second;
  hs_stream_t s = nullptr;
  const int dom = dev_dom_.count(device) ? dev_dom_.at(device) : 0;
  hs_ok(hs_stream_create(dctx_[size_t(dom)], 0, &s), "hs_stream_create");
  stream_dom_[s] = dom;
  sl.streams[key] = s;
  return s;
}

// Events are created in the domain of the stream they are recorded on: a
// component's events in its domain, the plan's fork (-1) on the origin, joins
// (-2, -3) with an explicit domain.
hs_event_t Engine::event(Slot& sl, int comp, int ev, int dom) {
  auto key = std::make_pair(comp, ev);
  auto it = sl.events.find(key);
  if (it != sl.events.end()) return it->second;
  if (dom < 0) dom = comp >= 0 && comp_dom_.count(comp) ? comp_dom_.at(comp) : 0;
  hs_event_t e = nullptr;
  hs_ok(hs_event_create(dctx_[size_t(dom)], 0, &e), "hs_event_create");
  sl.events[key] = e;
  return e;
}

// Whole-run graph over exactly one batch: per-instance inputs and outputs that are
// already dense in this GPU's memory are used in place. Every slot pointer inside
// such a group's / output's own allocation is redirected into the user's buffer at
// instance `first` (the layouts match: [batch][bytes]); the copy commands of those
// buffers are skipped during the capture. Not applied when an in-place input and
// output (or two outputs) overlap, or for io buffers (read and written by the DAG).
void Engine::zero_copy_remap(Slot& sl, int64_t first, int64_t n) {
  skip_groups_.clear();
  skip_outputs_.clear();
  if (!cfg_.zero_copy || n != cfg_.batch || dctx_.size() != 1) return;
  struct Range {
    char *lo, *hi, *to;
  };
  std::vector<Range> moves;
  std::vector<std::pair<char*, char*>> ins, outs;
  auto aligned = [](const char* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  for (size_t gi = 0; gi < groups_.size(); ++gi) {
    const Group& gr = groups_[gi];
    if (gr.resident || gr.io || !gr.b.on_device || gr.b.stride != gr.bytes || first + n > gr.b.count) continue;
    auto it = sl.group_buf.find({int(gi), 0});
    if (it == sl.group_buf.end()) continue;
    char* to = static_cast<char*>(gr.b.ptr) + first * gr.b.stride;
    if (!aligned(to)) continue;
    char* old = static_cast<char*>(it->second);
    moves.push_back({old, old + gr.bytes * n, to});
    ins.emplace_back(to, to + gr.bytes * n);
    skip_groups_.insert(int(gi));
  }
  for (const auto& key : outputs_) {
    const Binding& b = bindings_.at(key);
    const int64_t bytes = bytes_.at(key);
    if (!b.on_device || (b.stride != bytes && n > 1) || first + n > b.count || io_copy_.count(key)) continue;
    char* to = static_cast<char*>(b.ptr) + first * b.stride;
    if (!aligned(to)) continue;
    char* old = static_cast<char*>(sl.buf.at(key));
    moves.push_back({old, old + bytes * n, to});
    outs.emplace_back(to, to + bytes * n);
    skip_outputs_.insert(key);
  }
  auto overlap = [](const std::pair<char*, char*>& a, const std::pair<char*, char*>& b) {
    return a.first < b.second && b.first < a.second;
  };
  for (size_t i = 0; i < outs.size(); ++i) {
    for (const auto& r : ins)
      if (overlap(outs[i], r)) moves.clear();
    for (size_t j = i + 1; j < outs.size(); ++j)
      if (overlap(outs[i], outs[j])) moves.clear();
  }
  if (moves.empty()) {
    skip_groups_.clear();
    skip_outputs_.clear();
    return;
  }
  auto remap = [&](void*& p) {
    char* c = static_cast<char*>(p);
    for (const auto& m : moves)
      if (c >= m.lo && c < m.hi) {
        p = m.to + (c - m.lo);
        return;
      }
  };
  for (auto& [key, p] : sl.buf) remap(p);
  for (auto& [key, p] : sl.group_buf) remap(p);
}

void Engine::copy_in(Slot& sl, hs_stream_t s, int gi, int64_t first, int64_t n, int dom) {
  if (skip_groups_.count(gi)) return;  // read in place (zero_copy_remap)
  const Group& gr = groups_[size_t(gi)];
  auto dst = sl.group_buf.find({gi, dom});
  if (dst == sl.group_buf.end()) return;  // no kernel of this domain reads the group
  const char* src = static_cast<const char*>(gr.b.ptr) + first * gr.b.stride;
  hs_ok(hs_memcpy_2d(s, dst->second, size_t(gr.bytes), src, size_t(gr.b.stride), size_t(gr.bytes), size_t(n),
                     gr.b.on_device ? 2 : 0),
        "copy-in");
}

// Copy-in (in = true) or copy-out of one batch on the slot. With several memory
// domains each domain's copies run on its own copy stream, forked from and
// joined back into the origin stream.
void Engine::copies(Slot& sl, int64_t first, int64_t n, bool in) {
  if (dctx_.size() == 1) {
    if (in) {
      // independent input groups are copied side by side: group 0 on the origin
      // stream, the others on per-slot copy streams forked from and joined to it
      std::vector<int> gis;
      for (size_t gi = 0; gi < groups_.size(); ++gi)
        if (!groups_[gi].resident) gis.push_back(int(gi));
      if (gis.size() > 1) {
        if (!sl.copy_fork) hs_ok(hs_event_create(ctx_, 0, &sl.copy_fork), "hs_event_create");
        hs_ok(hs_event_record(sl.copy_fork, sl.origin), "copy fork");
      }
      for (size_t i = 0; i < gis.size(); ++i) {
        if (i == 0) {
          copy_in(sl, sl.origin, gis[i], first, n, 0);
          continue;
        }
        while (sl.copy_streams.size() < i) {
          hs_stream_t cs = nullptr;
          hs_event_t ce = nullptr;
          hs_ok(hs_stream_create(ctx_, 0, &cs), "hs_stream_create");
          hs_ok(hs_event_create(ctx_, 0, &ce), "hs_event_create");
          stream_dom_[cs] = 0;
          sl.copy_streams.push_back(cs);
          sl.copy_join.push_back(ce);
        }
        hs_stream_t cs = sl.copy_streams[i - 1];
        hs_ok(hs_stream_wait(cs, sl.copy_fork), "copy fork wait");
        copy_in(sl, cs, gis[i], first, n, 0);
        hs_ok(hs_event_record(sl.copy_join[i - 1], cs), "copy join");
        hs_ok(hs_stream_wait(sl.origin, sl.copy_join[i - 1]), "copy join wait");
      }
    } else {
      copy_out(sl, sl.origin, first, n, 0);
    }
    return;
  }
  hs_ok(hs_event_record(sl.copy_fork, sl.origin), "copy fork");
  for (size_t d = 0; d < dctx_.size(); ++d) {
    hs_stream_t s = dstream(sl, int(d));
    if (d > 0) hs_ok(hs_stream_wait(s, sl.copy_fork), "copy fork wait");
    if (in) {
      for (size_t gi = 0; gi < groups_.size(); ++gi)
        if (!groups_[gi].resident) copy_in(sl, s, int(gi), first, n, int(d));
    } else {
      copy_out(sl, s, first, n, int(d));
    }
    if (d > 0) {
      hs_event_t e = in ? sl.din.at(int(d)) : sl.dout.at(int(d));
      hs_ok(hs_event_record(e, s), "copy join");
      hs_ok(hs_stream_wait(sl.origin, e), "copy join wait");
    }
  }
}

void Engine::copy_out(Slot& sl, hs_stream_t s, int64_t first, int64_t n, int dom) {
  for (const auto& key : outputs_) {
    if (kdom(key.first) != dom || skip_outputs_.count(key)) continue;  // skipped: written in place
    const Binding& b = bindings_.at(key);
    const int64_t bytes = bytes_.at(key);
    char* dst = static_cast<char*>(b.ptr) + first * b.stride;
    hs_ok(hs_memcpy_2d(s, dst, size_t(b.stride ? b.stride : bytes), sl.buf.at(key), size_t(bytes), size_t(bytes),
                       size_t(b.stride ? n : 1), b.on_device ? 2 : 1),
          "copy-out");
  }
}

void Engine::launch_node(Slot& sl, hs_stream_t s, int kernel) {
  const Node& nd = nodes_.at(kernel);
  for (const auto& in : nd.inputs) {
    auto io = io_copy_.find(in);
    if (io != io_copy_.end())
      hs_ok(hs_memcpy_d2d(s, sl.buf.at(in), sl.buf.at(io->second), size_t(bytes_.at(in) * nb())), "io copy");
  }
  hs_op_args a{};
  a.n_in = int(nd.inputs.size());
  for (size_t i = 0; i < nd.inputs.size(); ++i) {
    const auto& key = nd.inputs[i];
    a.in[i] = sl.buf.at(key);
    auto gi = group_of_.find(key);
    const bool shared = gi != group_of_.end() && groups_[size_t(gi->second)].resident;
    a.in_stride[i] = shared ? 0 : bytes_.at(key) / 4;
  }
  a.out = static_cast<float*>(sl.buf.at(nd.output)) + nd.out_off;
  a.out_stride = bytes_.at(nd.output) / 4;
  for (int i = 0; i < 4; ++i) a.dims[i] = nd.dims[i];
  a.fparam[0] = nd.fparam[0];
  a.fparam[1] = nd.fparam[1];
  a.out_ld = nd.out_ld;
  a.epilogue = nd.epilogue;
  if (nd.epilogue == HS_EPI_SOFTMAX) a.fparam[0] = nd.escale;
  auto pl = node_planes_.find(kernel);
  a.aux = pl == node_planes_.end() ? nullptr : pl->second;
  if (nd.op == HS_OP_HEAD) {  // in = {X, Wh planes}, aux = Wq|Wk|Wv planes
    a.in[1] = a.aux;
    a.in_stride[1] = 0;
    a.aux = head_qkv_planes_.at(kernel);
  }
  a.flags = cfg_.deterministic ? HS_FLAG_DETERMINISTIC : 0;
  hs_ok(hs_launch(s, nd.op, &a, cfg_.math, int(nb())), "hs_launch");
}

void Engine::issue(Slot& sl, const TaskComponent& t, const CommandQueueStructure& q, int prev_comp,
                   const CommandQueueStructure* prev_q, bool graph, int64_t first, int64_t n) {
  const int d = q.device;
  std::set<int> dep_sources;
  std::map<int, std::vector<int>> preds;
  for (auto [a, b] : q.deps) {
    dep_sources.insert(a);
    preds[b].push_back(a);
  }
  // Device exclusivity in graph mode: every queue waits for the previous
  // component's terminal commands on this logical device.
  if (prev_q) {
    for (size_t qi = 0; qi < q.queues.size(); ++qi) {
      if (q.queues[qi].empty()) continue;
      hs_stream_t s = stream(sl, d, int(qi));
      for (int te : prev_q->terminal_events()) hs_ok(hs_stream_wait(s, event(sl, prev_comp, te)), "exclusivity wait");
    }
  }
  // Commands in global enqueue order: every E_Q / inter-edge source is
  // recorded on the host before any stream waits on it.
  for (int ev = 0; ev < q.event_count; ++ev) {
    const auto [qi, idx] = q.event_pos[size_t(ev)];
    const Command& c = q.queues[size_t(qi)][size_t(idx)];
    hs_stream_t s = stream(sl, d, qi);
    auto pit = preds.find(ev);
    if (pit != preds.end())
      for (int p : pit->second) hs_ok(hs_stream_wait(s, event(sl, t.id, p)), "E_Q wait");
    bool record = dep_sources.count(ev) || q.callbacks.count(ev);
    TraceRec tr;
    if (tracing_) {
      tr.component = t.id;
      tr.event = ev;
      tr.kind = int(c.kind);
      tr.kernel = c.kernel;
      tr.device = d;
      tr.queue = qi;
      tr.label = c.label;
      hs_ctx_t tctx = dctx_[size_t(stream_dom_.count(s) ? stream_dom_.at(s) : 0)];
      hs_ok(hs_event_create(tctx, 1, &tr.t0), "hs_event_create");
      hs_ok(hs_event_create(tctx, 1, &tr.t1), "hs_event_create");
      hs_ok(hs_event_record(tr.t0, s), "trace record");
    }
    switch (c.kind) {
      case CmdKind::write: {
        const std::pair<int, int> key{c.buffer->kernel, c.buffer->pos};
        if (c.dependent) {
          auto src = sl.edge_event.find(c.edge);
          if (src == sl.edge_event.end())
            fail(Errc::deadlock, "dependent write for edge " + std::to_string(c.edge) + " issued before its producer");
          hs_ok(hs_stream_wait(s, event(sl, src->second.first, src->second.second)), "inter-edge wait");
          auto io = io_copy_.find(key);
          auto pr = peer_in_.find(key);
          if (io != io_copy_.end())
            hs_ok(hs_memcpy_d2d(s, sl.buf.at(key), sl.buf.at(io->second), size_t(bytes_.at(key) * nb())),
                  "dependent write");
          else if (pr != peer_in_.end())  // producer in another memory domain: one peer copy (NVLink)
            hs_ok(hs_memcpy_peer(s, sl.buf.at(key), dom_gpu_[size_t(kdom(key.first))], sl.buf.at(pr->second),
                                 dom_gpu_[size_t(kdom(pr->second.first))], size_t(bytes_.at(key) * nb())),
                  "dependent write (peer)");
        } else if (!graph) {
          const int gi = group_of_.at(key);
          if (!groups_[size_t(gi)].resident) {
            if (!sl.group_done.count(gi)) {
              copy_in(sl, s, gi, first, n, 0);
              auto ge = sl.group_event.find(gi);
              hs_event_t e = nullptr;
              if (ge == sl.group_event.end()) {
                hs_ok(hs_event_create(ctx_, 0, &e), "hs_event_create");
                sl.group_event[gi] = e;
              } else {
                e = ge->second;
              }
              hs_ok(hs_event_record(e, s), "group record");
              sl.group_done.insert(gi);
            } else {
              hs_ok(hs_stream_wait(s, sl.group_event.at(gi)), "group wait");
            }
          }
        }
        break;
      }
      case CmdKind::ndrange: {
        const bool fused = graph || dyn_fused_;
        auto lead = fused ? fuse_leader_.find({t.id, ev}) : fuse_leader_.end();
        auto member = fused ? fuse_member_.find({t.id, ev}) : fuse_member_.end();
        if (lead != fuse_leader_.end()) {
          // Grouped launch for every member: first make this stream wait for the
          // other members' inter-edge inputs (their dependent writes come later
          // in enqueue order), then one tcgen05 launch writes all outputs.
          const FuseGroup& fg = fuse_groups_[size_t(lead->second)];
          for (size_t m = 1; m < fg.kernels.size(); ++m)
            for (const auto& qq : q.queues)
              for (const Command& w : qq)
                if (w.kernel == fg.kernels[m] && w.kind == CmdKind::write && w.dependent) {
                  auto src = sl.edge_event.find(w.edge);
                  if (src == sl.edge_event.end()) fail(Errc::deadlock, "grouped launch before its producer");
                  hs_ok(hs_stream_wait(s, event(sl, src->second.first, src->second.second)), "inter-edge wait");
                }
          if (fg.absorbed) {  // computed by the whole-head launch of this component
            record = true;
            break;
          }
          const Node& nd = nodes_.at(fg.kernels[0]);
          hs_op_args a{};
          a.n_in = 2;
          a.in[0] = sl.buf.at(nd.inputs[0]);
          {  // a resident A (one shared copy) is read by every instance: stride 0
            auto agi = group_of_.find(nd.inputs[0]);
            const bool shared = agi != group_of_.end() && groups_[size_t(agi->second)].resident;
            a.in_stride[0] = shared ? 0 : bytes_.at(nd.inputs[0]) / 4;
          }
          a.in[1] = sl.buf.at(nd.inputs[1]);
          a.in_stride[1] = 0;
          a.out = sl.buf.at(nd.output);
          a.out_stride = bytes_.at(nd.output) / 4;
          for (int i = 0; i < 3; ++i) a.dims[i] = nd.dims[i];
          a.aux = fg.planes;
          a.n_out = int(fg.kernels.size());
          for (size_t m = 0; m < fg.kernels.size(); ++m) {
            const auto& okey = nodes_.at(fg.kernels[m]).output;
            a.outs[m] = sl.buf.at(okey);
            a.out_strides[m] = bytes_.at(okey) / 4;
          }
          a.flags = cfg_.deterministic ? HS_FLAG_DETERMINISTIC : 0;
          hs_ok(hs_launch(s, nd.op, &a, cfg_.math, int(nb())), "hs_launch (grouped)");
          record = true;
        } else if (member != fuse_member_.end()) {
          // computed by the group's leader launch: order this queue after it
          const FuseGroup& fg = fuse_groups_[size_t(member->second)];
          hs_ok(hs_stream_wait(s, event(sl, t.id, fg.events[0])), "grouped member wait");
        } else if (!nodes_.at(c.kernel).elided) {
          launch_node(sl, s, c.kernel);
        }  // elided: computed by the launch that absorbed it (plan_chain_rewrites)
        break;
      }
      case CmdKind::read:
        if (c.dependent) {
          sl.edge_event[c.edge] = {t.id, ev};
          record = true;
        } else if (!graph) {
          const std::pair<int, int> key{c.buffer->kernel, c.buffer->pos};
          if (bindings_.count(key)) {
            const Binding& b = bindings_.at(key);
            const int64_t bytes = bytes_.at(key);
            hs_ok(hs_memcpy_2d(s, static_cast<char*>(b.ptr) + first * b.stride, size_t(b.stride ? b.stride : bytes),
                               sl.buf.at(key), size_t(bytes), size_t(bytes), size_t(b.stride ? n : 1),
                               b.on_device ? 2 : 1),
                  "isolated read");
          }
        }
        break;
    }
    if (tracing_) {
      hs_ok(hs_event_record(tr.t1, s), "trace record");
      trace_.push_back(tr);
    }
    if (record) hs_ok(hs_event_record(event(sl, t.id, ev), s), "event record");
    if (!graph && q.callbacks.count(ev))
      hs_ok(hs_host_callback(s, &CUDART_CB_trampoline, new_callback({t.id, ev})), "host callback");
  }
}

void Engine::plan_fusion() {
  auto producers = g_.producer_edge();
  const auto& ec = sched_->edge_classes();
  for (const auto& q : plan_.structures) {
    std::set<int> dep_targets;
    for (auto [a, b] : q.deps) dep_targets.insert(b);
    // candidate key: (op, resolved A source, M, N, K) -> ndrange events
    std::map<std::tuple<int, long long, int64_t, int64_t, int64_t>, std::vector<std::pair<int, int>>> cands;
    for (int ev = 0; ev < q.event_count; ++ev) {
      const Command& c = q.command_of(ev);
      if (c.kind != CmdKind::ndrange || dep_targets.count(ev)) continue;
      const Node& nd = nodes_.at(c.kernel);
      if ((nd.op != HS_OP_GEMM && nd.op != HS_OP_GEMM_RELU) || !node_planes_.count(c.kernel)) continue;
      if (nd.dims[1] != 64) continue;  // grouped tiles of 2 x 64 or 3 x 64 columns
      // no producer inside the component: launching early cannot reorder a data dependency
      bool intra = false;
      for (const auto& in : nd.inputs) {
        auto pe = producers.find(in);
        if (pe != producers.end() && ec.edge_kind[size_t(pe->second)] == EdgeKind::intra) intra = true;
      }
      if (intra) continue;
      const auto& a = nd.inputs[0];
      long long src;
      auto al = alias_.find(a);
      if (al != alias_.end()) src = (static_cast<long long>(al->second.first) << 20) | al->second.second;
      else if (group_of_.count(a)) src = -1 - group_of_.at(a);
      else continue;
      cands[{nd.op, src, nd.dims[0], nd.dims[1], nd.dims[2]}].push_back({ev, c.kernel});
    }
    for (auto& [key, list] : cands) {
      size_t i = 0;
      while (list.size() - i >= 2) {
        const size_t take = (list.size() - i) >= 3 ? 3 : 2;
        FuseGroup fg;
        fg.component = q.component;
        fg.n = std::get<3>(key);
        fg.k = std::get<4>(key);
        for (size_t j = 0; j < take; ++j) {
          fg.events.push_back(list[i + j].first);
          fg.kernels.push_back(list[i + j].second);
        }
        fg.planes = dalloc(comp_dom_.count(q.component) ? comp_dom_.at(q.component) : 0,
                           2 * int64_t(take) * fg.n * fg.k * plane_elem_bytes());
        const int gi = int(fuse_groups_.size());
        fuse_leader_[{q.component, fg.events[0]}] = gi;
        for (size_t j = 1; j < take; ++j) fuse_member_[{q.component, fg.events[j]}] = gi;
        launches_per_batch_ -= int64_t(take) - 1;
        fuse_groups_.push_back(std::move(fg));
        i += take;
      }
    }
  }
}

// Chain rewrites (graph mode). Each rule removes one node's launch by folding
// it into its producer; it fires only when the intermediate buffer is
// internal to the DAG (exactly one consumer edge, no isolated read), so no
// observable buffer changes. The plan's commands, events and E_Q / inter-edge
// waits are untouched: an elided ndrange still records its events, so every
// consumer keeps waiting on the same chain.
//   transpose_into_gemm_nt  T = transpose(X) consumed only as B of a gemm:
//                           the gemm reads X as gemm_nt (B = [N,K]).
//   softmax_epilogue        P = softmax(S·s) where S = gemm(..) feeds only the
//                           softmax and N <= 128: the gemm computes P directly.
//   concat_in_place         Y = concat(Z_0..Z_n-1), Z_i = gemm(..) feeding only
//                           the concat: gemm i writes Y[:, i·c:(i+1)·c] (ld n·c).
void Engine::plan_chain_rewrites() {
  const auto consumers = g_.consumer_edges();
  std::set<int> grouped;
  for (const auto& fg : fuse_groups_) grouped.insert(fg.kernels.begin(), fg.kernels.end());
  auto sole_consumer = [&](std::pair<int, int> out, int* dst_kernel, int* dst_pos) {
    auto it = consumers.find(out);
    if (it == consumers.end() || it->second.size() != 1) return false;
    const DagEdge& e = g_.edges[size_t(it->second.front())];
    if (io_copy_.count({e.dst_kernel, e.dst_pos})) return false;  // io inputs are copies, not aliases
    // an edge between memory domains is a peer copy: no rewrite may let one side
    // address the other side's buffer directly
    if (peer_in_.count({e.dst_kernel, e.dst_pos}) || kdom(e.src_kernel) != kdom(e.dst_kernel)) return false;
    *dst_kernel = e.dst_kernel;
    *dst_pos = e.dst_pos;
    return true;
  };
  auto is_gemm = [](int op) { return op == HS_OP_GEMM || op == HS_OP_GEMM_NT || op == HS_OP_GEMM_RELU; };
  auto resident = [&](std::pair<int, int> key) {
    auto gi = group_of_.find(key);
    return gi != group_of_.end() && groups_[size_t(gi->second)].resident;
  };
  for (auto& [kid, nd] : nodes_) {
    if (nd.op != HS_OP_TRANSPOSE || nd.elided) continue;
    int ck, cp;
    if (!sole_consumer(nd.output, &ck, &cp)) continue;
    Node& g = nodes_.at(ck);
    if (g.op != HS_OP_GEMM || cp != g.inputs[1].second || grouped.count(ck) || g.epilogue) continue;
    if (resident(nd.inputs[0]) || node_planes_.count(ck)) continue;
    // X is R x C; T = X^T is C x R = K x N, so gemm_nt reads X as [N = R, K = C]
    if (g.dims[1] != nd.dims[0] || g.dims[2] != nd.dims[1]) continue;
    g.op = HS_OP_GEMM_NT;
    g.inputs[1] = nd.inputs[0];
    nd.elided = true;
    ++rewrites_["transpose_into_gemm_nt"];
  }
  // scale_into_softmax: B = scale(A, s) consumed only by P = softmax(B, t): the
  // softmax reads A with scale s·t (one rounding instead of two; within
  // tolerance, not bit-identical to the two launches).
  std::map<int, int> folded_scale;  // elided scale -> the softmax that absorbed it
  for (auto& [kid, sc] : nodes_) {
    if (sc.op != HS_OP_SCALE || sc.elided) continue;
    int ck, cp;
    if (!sole_consumer(sc.output, &ck, &cp)) continue;
    Node& sm = nodes_.at(ck);
    if (sm.op != HS_OP_SOFTMAX || sm.elided || sc.dims[0] != sm.dims[0] * sm.dims[1] || resident(sc.inputs[0]))
      continue;
    sm.inputs[0] = sc.inputs[0];
    sm.fparam[0] *= sc.fparam[0];
    sc.elided = true;
    folded_scale[kid] = ck;
    ++rewrites_["scale_into_softmax"];
  }
  for (auto& [kid, g] : nodes_) {
    if ((g.op != HS_OP_GEMM && g.op != HS_OP_GEMM_NT) || g.elided || g.epilogue || grouped.count(kid)) continue;
    int ck, cp;
    if (!sole_consumer(g.output, &ck, &cp)) continue;
    if (folded_scale.count(ck)) ck = folded_scale.at(ck);  // gemm -> (scale folded into) softmax
    Node& sm = nodes_.at(ck);
    if (sm.op != HS_OP_SOFTMAX || sm.elided) continue;
    if (sm.dims[0] != g.dims[0] || sm.dims[1] != g.dims[1] || g.dims[1] > 128) continue;
    g.epilogue = HS_EPI_SOFTMAX;
    g.escale = sm.fparam[0];
    g.output = sm.output;
    sm.elided = true;
    ++rewrites_["softmax_epilogue"];
  }
  for (auto& [kid, cat] : nodes_) {
    if (cat.op != HS_OP_CONCAT || cat.elided) continue;
    const int64_t n = int64_t(cat.inputs.size()), rows = cat.dims[0], cols = cat.dims[1];
    std::vector<int> producers;
    for (const auto& in : cat.inputs) {
      auto al = alias_.find(in);
      if (al == alias_.end()) break;
      int ck, cp;
      if (!sole_consumer(al->second, &ck, &cp) || ck != kid) break;
      const int pk = al->second.first;
      const Node& z = nodes_.at(pk);
      if (!is_gemm(z.op) || z.elided || grouped.count(pk) || z.out_ld || z.output != al->second) break;
      if (z.dims[0] != rows || z.dims[1] != cols) break;
      producers.push_back(pk);
    }
    if (int64_t(producers.size()) != n || cols % 4) continue;
    for (int64_t i = 0; i < n; ++i) {
      Node& z = nodes_.at(producers[size_t(i)]);
      z.output = cat.output;
      z.out_off = i * cols;
      z.out_ld = n * cols;
    }
    cat.elided = true;
    ++rewrites_["concat_in_place"];
  }
  // attention_head: P = gemm_nt(Q, K) with the softmax epilogue (rules above),
  // C = gemm(P, V), Z = gemm(C, W) with W resident, each intermediate feeding
  // only the next: one HS_OP_ATTN_HEAD launch computes Z (keeping any concat
  // placement of Z); the first two GEMMs are elided.
  for (auto& [kid, z] : nodes_) {
    if (z.op != HS_OP_GEMM || z.elided || z.epilogue || grouped.count(kid) || !resident(z.inputs[1])) continue;
    auto pc = alias_.find(z.inputs[0]);
    if (pc == alias_.end()) continue;
    int ck, cp;
    if (!sole_consumer(pc->second, &ck, &cp) || ck != kid) continue;
    const int k2 = pc->second.first;
    Node& g2 = nodes_.at(k2);
    if (g2.op != HS_OP_GEMM || g2.elided || g2.epilogue || g2.out_ld || grouped.count(k2) || g2.output != pc->second)
      continue;
    if (resident(g2.inputs[1])) continue;  // V is an activation
    auto pp = alias_.find(g2.inputs[0]);
    if (pp == alias_.end() || !sole_consumer(pp->second, &ck, &cp) || ck != k2) continue;
    // P is the softmax node's output, written by the GEMM that absorbed it
    int k1 = -1;
    for (const auto& [id, nd] : nodes_)
      if (!nd.elided && nd.op == HS_OP_GEMM_NT && nd.epilogue == HS_EPI_SOFTMAX && nd.output == pp->second) k1 = id;
    if (k1 < 0 || grouped.count(k1)) continue;
    Node& g1 = nodes_.at(k1);
    const int64_t S = g1.dims[0];
    if (g1.dims[1] != S || g1.dims[2] != 64 || g1.out_ld || S > 128) continue;
    if (g2.dims[0] != S || g2.dims[1] != 64 || g2.dims[2] != S) continue;
    if (z.dims[0] != S || z.dims[1] != 64 || z.dims[2] != 64) continue;
    const std::pair<int, int> wkey = z.inputs[1];
    z.op = HS_OP_ATTN_HEAD;
    z.inputs = {g1.inputs[0], g1.inputs[1], g2.inputs[1], wkey};
    z.dims[0] = S;
    z.dims[1] = 64;
    z.dims[2] = 64;
    z.fparam[0] = g1.escale;
    g1.elided = true;
    g2.elided = true;
    if (plane_format() != 0) {  // the fused head consumes tf32 planes; BF16X3 keeps bf16 ones for GEMMs
      const int gi = group_of_.at(wkey);
      const int dom = kdom(kid);
      auto it = attn_planes_.find({gi, dom});
      if (it == attn_planes_.end()) {
        Planes pl;
        pl.gi = gi;
        pl.n = 64;
        pl.k = 64;
        pl.dom = dom;
        pl.ptr = dalloc(dom, 2 * 64 * 64 * 4);
        it = attn_planes_.emplace(std::make_pair(gi, dom), pl).first;
      }
      node_planes_[kid] = it->second.ptr;
    }
    ++rewrites_["attention_head"];
  }
  // head_fused: an attn_head whose Q, K, V are the three outputs of one grouped
  // projection launch (shared X, resident tf32 planes), each feeding only this
  // node: one HS_OP_HEAD launch computes Z from X and the grouped launch is
  // absorbed (its commands and events stay; only its kernel is not launched).
  if (cfg_.fuse >= 3 && plane_format() == 0) {
    for (auto& [kid, z] : nodes_) {
      if (z.op != HS_OP_ATTN_HEAD || z.elided) continue;
      int prod[3] = {-1, -1, -1};
      bool ok = true;
      for (int i = 0; i < 3 && ok; ++i) {
        auto al = alias_.find(z.inputs[size_t(i)]);
        int ck, cp;
        // the producer's single consumer edge goes to z or to a node absorbed into z
        // (the elided gemm_nt / transpose / P·V GEMM of the attention_head rule)
        if (al == alias_.end() || !sole_consumer(al->second, &ck, &cp) || (ck != kid && !nodes_.at(ck).elided)) {
          ok = false;
          break;
        }
        const Node& pn = nodes_.at(al->second.first);
        if (pn.op != HS_OP_GEMM || pn.elided || pn.epilogue || pn.out_ld || pn.output != al->second ||
            pn.dims[0] != z.dims[0] || pn.dims[1] != 64 || pn.dims[2] % 32)
          ok = false;
        prod[i] = al->second.first;
      }
      if (!ok) continue;
      FuseGroup* fg = nullptr;
      for (auto& g : fuse_groups_) {
        if (g.absorbed || g.kernels.size() != 3) continue;
        std::set<int> members(g.kernels.begin(), g.kernels.end());
        if (members == std::set<int>{prod[0], prod[1], prod[2]}) fg = &g;
      }
      // the members read one X (plan_fusion grouped them by resolved A source)
      if (!fg || fg->n != 64) continue;
      fg->kernels = {prod[0], prod[1], prod[2]};  // plane order q | k | v (the leader event is unchanged)
      fg->absorbed = true;
      const std::pair<int, int> wkey = z.inputs[3];
      z.op = HS_OP_HEAD;
      z.inputs = {nodes_.at(prod[0]).inputs[0], wkey};
      z.dims[1] = fg->k;
      z.dims[2] = 64;
      head_qkv_planes_[kid] = fg->planes;
      --launches_per_batch_;
      ++rewrites_["head_fused"];
    }
  }
  for (const auto& [kid, nd] : nodes_)
    if (nd.elided) --launches_per_batch_;
}

void Engine::emit_plan(Slot& sl) {
  // Every stream the plan touches joins through a fork event on the origin
  // stream and is joined back at the end (the capture boundary in graph mode).
  std::set<std::pair<int, int>> used;
  for (size_t i = 0; i < plan_.dispatches.size(); ++i) {
    const auto& q = plan_.structures[i];
    for (size_t qi = 0; qi < q.queues.size(); ++qi) used.insert({q.device, int(qi)});
  }
  hs_event_t fork = event(sl, -1, 0);
  hs_ok(hs_event_record(fork, sl.origin), "fork record");
  for (auto [d, qi] : used) hs_ok(hs_stream_wait(stream(sl, d, qi), fork), "fork wait");
  std::map<int, int> last_on_device;  // logical device -> index into plan_
  for (size_t i = 0; i < plan_.dispatches.size(); ++i) {
    const auto& rec = plan_.dispatches[i];
    const auto& q = plan_.structures[i];
    auto prev = last_on_device.find(rec.device);
    const CommandQueueStructure* pq = prev == last_on_device.end() ? nullptr : &plan_.structures[size_t(prev->second)];
    int pc = prev == last_on_device.end() ? -1 : plan_.dispatches[size_t(prev->second)].component;
    issue(sl, sched_->components()[size_t(rec.component)], q, pc, pq, true, 0, cfg_.batch);
    last_on_device[rec.device] = int(i);
  }
  int j = 0;
  for (auto [d, qi] : used) {
    hs_event_t e = event(sl, -2, j++, dev_dom_.count(d) ? dev_dom_.at(d) : 0);
    hs_ok(hs_event_record(e, stream(sl, d, qi)), "join record");
    hs_ok(hs_stream_wait(sl.origin, e), "join wait");
  }
}

void Engine::capture(Slot& sl) {
  for (size_t i = 0; i < plan_.dispatches.size(); ++i) {
    const auto& q = plan_.structures[i];
    for (size_t qi = 0; qi < q.queues.size(); ++qi) stream(sl, q.device, int(qi));  // create before capture
  }
  hs_ok(hs_capture_begin(sl.origin), "capture begin");
  emit_plan(sl);
  hs_ok(hs_capture_end(sl.origin, &sl.graph), "capture end");
  if (ramp_ > 0) {  // the same plan for ramp_ instances (first and last chunks of a host-fed stream)
    cur_batch_ = ramp_;
    hs_ok(hs_capture_begin(sl.origin), "capture begin");
    emit_plan(sl);
    hs_ok(hs_capture_end(sl.origin, &sl.graph_small), "capture end");
    cur_batch_ = 0;
  }
}

void Engine::clear_trace() {
  for (auto& r : trace_) {
    hs_event_destroy(r.t0);
    hs_event_destroy(r.t1);
  }
  trace_.clear();
  trace_dispatch_.clear();
}

void* Engine::new_callback(const Completion& c) {
  std::lock_guard<std::mutex> lk(mu_);
  return new CbData{this, c};
}

// Notified under the lock: once this thread releases mu_ it no longer touches the
// engine, so the scheduler thread may finish the run and destroy it (ThreadSanitizer
// caught the notify-after-unlock variant racing ~Engine's pthread_cond_destroy).
void Engine::deliver_callback(void* p) {
  auto* d = static_cast<CbData*>(p);
  std::lock_guard<std::mutex> lk(mu_);
  done_q_.push_back(d->c);
  pending_.fetch_add(1, std::memory_order_release);
  delete d;
  cv_.notify_one();
}

void Engine::push_completion(const Completion& c) {
  std::lock_guard<std::mutex> lk(mu_);
  done_q_.push_back(c);
  pending_.fetch_add(1, std::memory_order_release);
  cv_.notify_one();
}

// The scheduler thread spins on the completion count for a short while before
// sleeping on the condition variable: a host callback usually arrives within
// tens of microseconds, and a condition-variable wake-up would add about as much.
Completion Engine::wait_completion() {
  const auto t0 = std::chrono::steady_clock::now();
  while (pending_.load(std::memory_order_acquire) == 0 &&
         std::chrono::steady_clock::now() - t0 < std::chrono::microseconds(kSpinUs)) {
  }
  std::unique_lock<std::mutex> lk(mu_);
  if (!cv_.wait_for(lk, std::chrono::seconds(120), [&] { return !done_q_.empty(); }))
    fail(Errc::deadlock, "no completion callback within 120 s");
  Completion c = done_q_.front();
  done_q_.pop_front();
  pending_.fetch_sub(1, std::memory_order_relaxed);
  last_log_.push_back(c);
  host_wait_ns_ += std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
  return c;
}

void Engine::reset_dynamic_state(Slot& sl) {
  sl.group_done.clear();
  sl.edge_event.clear();
  last_log_.clear();
  std::lock_guard<std::mutex> lk(mu_);
  done_q_.clear();
  pending_.store(0, std::memory_order_relaxed);
}

void Engine::run_dynamic(Slot& sl, int64_t first, int64_t n) {
  reset_dynamic_state(sl);
  ext_first_ = first;
  ext_n_ = n;
  CudaDispatch ex(*this);
  ScheduleResult r = sched_->run(ex);
  last_dispatches_ = r.dispatches;
  if (tracing_)
    for (const auto& rec : r.dispatches) trace_dispatch_.push_back({rec.component, rec.device});
}

void Engine::ext_dispatch(const TaskComponent& t, const CommandQueueStructure& q) {
  if (cfg_.graph_mode) fail(Errc::invalid_param, "external dispatch needs a dynamic-mode engine");
  const auto t0 = std::chrono::steady_clock::now();
  issue(slots_.front(), t, q, -1, nullptr, false, ext_first_, ext_n_);
  host_dispatch_ns_ +=
      std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
  ++host_dispatches_;
}

Completion Engine::ext_wait() { return wait_completion(); }

void Engine::check_range(int64_t first, int64_t n) const {
  if (n < 1) fail(Errc::invalid_param, "n_instances must be >= 1");
  if (first < 0) fail(Errc::invalid_param, "first must be >= 0");
  for (const auto& [key, b] : bindings_)
    if (b.stride > 0 && first + n > b.count)
      fail(Errc::invalid_param, "instances [" + std::to_string(first) + ", " + std::to_string(first + n) +
                                    ") exceed the " + std::to_string(b.count) + " bound at (" +
                                    std::to_string(key.first) + "," + std::to_string(key.second) + ")");
}

void Engine::join_dynamic_streams(Slot& s0) {
  int j = 0;
  for (auto& [k, s] : s0.streams) {
    hs_event_t e = event(s0, -3, j++);
    hs_ok(hs_event_record(e, s), "join record");
    hs_ok(hs_stream_wait(s0.origin, e), "join wait");
  }
}

// A caller-driven run: the caller's scheduler dispatches each component of one
// batch of n instances through ext_dispatch and drains completions with ext_wait.
void Engine::ext_begin(int64_t first, int64_t n) {
  if (cfg_.graph_mode) fail(Errc::invalid_param, "external dispatch needs a dynamic-mode engine");
  if (ext_open_) fail(Errc::invalid_param, "begin() called twice without end()");
  check_range(first, n);
  if (n > cfg_.batch) fail(Errc::invalid_param, "n exceeds the executor's batch");
  plan_once();
  upload_resident();
  Slot& s0 = slots_.front();
  reset_dynamic_state(s0);
  ext_first_ = first;
  ext_n_ = n;
  hs_ok(hs_event_record(s0.t_start, s0.origin), "start record");
  for (auto& [k, s] : s0.streams) hs_ok(hs_stream_wait(s, s0.t_start), "start wait");
  ext_open_ = true;
}

int64_t Engine::ext_end() {
  if (!ext_open_) fail(Errc::invalid_param, "end() without begin()");
  ext_open_ = false;
  Slot& s0 = slots_.front();
  join_dynamic_streams(s0);
  hs_ok(hs_event_record(s0.t_end, s0.origin), "end record");
  hs_ok(hs_event_sync(s0.t_end), "end sync");
  int64_t ns = 0;
  hs_ok(hs_event_elapsed_ns(s0.t_start, s0.t_end, &ns), "elapsed");
  ++runs_;
  ++batches_run_;
  return ns;
}

void Engine::plan_once() {
  if (planned_) return;
  // Dynamic mode launches one kernel per ndrange, unless dynamic_fuse asks for the
  // graph plan's launch lowering: the rewrites are per component and keyed by
  // (component, event), and setup_cq numbers a component's events the same on
  // every device when all devices have the same queue count.
  bool uniform_queues = true;
  for (const auto& d : platform_.devices) uniform_queues = uniform_queues && d.queues == platform_.devices[0].queues;
  if (!cfg_.graph_mode && cfg_.dynamic_fuse && (!uniform_queues || cfg_.math == HS_MATH_FP32_SIMT))
    fail(Errc::invalid_param, uniform_queues ? "dynamic_fuse needs tcgen05 math (not simt)"
                                             : "dynamic_fuse needs the same queue count on every device");
  dyn_fused_ = !cfg_.graph_mode && cfg_.dynamic_fuse;
  if (cfg_.graph_mode || dyn_fused_) {
    PlanExecutor pe;
    plan_ = sched_->run(pe);
    place_components();
  }
  plan_buffers();
  if (dyn_fused_) {
    if (cfg_.fuse >= 1) plan_fusion();
    if (cfg_.fuse >= 2) plan_chain_rewrites();
  }
  if (cfg_.graph_mode) {
    if (cfg_.fuse >= 1 && cfg_.math != HS_MATH_FP32_SIMT) plan_fusion();
    if (cfg_.fuse >= 2 && cfg_.math != HS_MATH_FP32_SIMT) plan_chain_rewrites();
  }
  place_slot_buffers();
  if (cfg_.graph_mode) {
    // Ramp (host-fed streams): the first and last chunks of a run are ramp_ =
    // batch/4 instances, so the copy-in before the first graph and the copy-out
    // after the last one are short; the copies of every other chunk overlap
    // the graphs of the other slots.
    bool host_io = false;
    for (const auto& gr : groups_)
      if (!gr.resident && !gr.b.on_device) host_io = true;
    for (const auto& key : outputs_)
      if (!bindings_.at(key).on_device) host_io = true;
    if (cfg_.ramp && host_io && !cfg_.trace && cfg_.batch >= 8 && slots_.size() > 1)
      ramp_ = cfg_.ramp > 1 ? std::min<int64_t>(cfg_.ramp, cfg_.batch / 2) : cfg_.batch / 4;
    if (capture_ok_)
      for (auto& sl : slots_) capture(sl);
  }
  planned_ = true;
}

void Engine::run(int64_t first, int64_t n, int64_t* elapsed_ns) {
  check_range(first, n);
  if (ext_open_) fail(Errc::invalid_param, "run() inside an open begin()/end() pair");
  plan_once();
  upload_resident();
  const int64_t B = cfg_.batch;
  const int64_t nb = (n + B - 1) / B;
  Slot& s0 = slots_.front();
  // Every stream that can carry work starts after t_start.
  hs_ok(hs_event_record(s0.t_start, s0.origin), "start record");
  for (size_t i = 1; i < slots_.size(); ++i) hs_ok(hs_stream_wait(slots_[i].origin, s0.t_start), "start wait");
  if (cfg_.trace) clear_trace();
  if (cfg_.graph_mode) {
    // chunks of the stream: (offset, count, small graph?)
    std::vector<std::tuple<int64_t, int64_t, bool>> chunks;
    if (ramp_ > 0 && capture_ok_ && n >= 4 * B) {
      const int64_t R = ramp_;
      const int64_t full = (n - 2 * R) / B;
      int64_t off = 0;
      chunks.emplace_back(off, R, true);
      off += R;
      for (int64_t i = 0; i < full; ++i, off += B) chunks.emplace_back(off, B, false);
      for (; off < n; off += R) chunks.emplace_back(off, std::min(R, n - off), true);
    } else {
      for (int64_t b = 0; b < nb; ++b) chunks.emplace_back(b * B, std::min(B, n - b * B), false);
    }
    const int64_t n_chunks = int64_t(chunks.size());
    // A run that is one chunk (the latency configs: one DAG, or one batch of them)
    // replays a graph that also holds its copies: one host submission per run instead
    // of the copy commands, their fork/join events and the plan launch. Bindings are
    // frozen after planning, so the graph stays valid for this (first, n) window.
    if (chunks.size() == 1 && capture_ok_ && !cfg_.trace && dctx_.size() == 1 && cfg_.run_graph) {
      Slot& sl = slots_.front();
      if (!sl.graph_run || sl.run_first != first || sl.run_n != n) {
        hs_graph_destroy(sl.graph_run);
        sl.graph_run = nullptr;
        // the slot's own pointers come back however the capture ends (a failed launch
        // throws out of emit_plan)
        struct Restore {
          Engine* e;
          Slot& sl;
          decltype(sl.buf) buf;
          decltype(sl.group_buf) group_buf;
          ~Restore() {
            sl.buf = std::move(buf);
            sl.group_buf = std::move(group_buf);
            e->skip_groups_.clear();
            e->skip_outputs_.clear();
          }
        } restore{this, sl, sl.buf, sl.group_buf};
        zero_copy_remap(sl, first, n);
        zero_copy_groups_ = int64_t(skip_groups_.size());
        zero_copy_outputs_ = int64_t(skip_outputs_.size());
        hs_ok(hs_capture_begin(sl.origin), "capture begin");
        copies(sl, first, n, true);
        emit_plan(sl);
        copies(sl, first, n, false);
        hs_ok(hs_capture_end(sl.origin, &sl.graph_run), "capture end");
        sl.run_first = first;
        sl.run_n = n;
      }
      hs_ok(hs_graph_launch(sl.graph_run, sl.origin), "graph launch");
      chunks.clear();
    }
    for (size_t ci = 0; ci < chunks.size(); ++ci) {
      const auto [off, cnt, small] = chunks[ci];
      const int64_t b = int64_t(ci);
      Slot& sl = slots_[size_t(b % int64_t(slots_.size()))];
      const int64_t f = first + off;
      copies(sl, f, cnt, true);
      if ((cfg_.trace && b == 0) || !capture_ok_) {
        // traced batch: the same plan issued directly (not replayed) with a
        // timing event pair around every command
        // (or: several GPUs, where the plan is issued directly every batch)
        tracing_ = cfg_.trace && b == 0;
        if (tracing_)
          for (const auto& rec : plan_.dispatches) trace_dispatch_.push_back({rec.component, rec.device});
        emit_plan(sl);
        tracing_ = false;
      } else {
        hs_ok(hs_graph_launch(small ? sl.graph_small : sl.graph, sl.origin), "graph launch");
      }
      copies(sl, f, cnt, false);
    }
    batches_run_ += n_chunks - nb;  // counted below as nb
  } else {
    for (auto& [k, s] : s0.streams) hs_ok(hs_stream_wait(s, s0.t_start), "start wait");
    for (int64_t b = 0; b < nb; ++b) {
      const int64_t f = first + b * B, cnt = std::min(B, n - b * B);
      tracing_ = cfg_.trace && b == 0;
      run_dynamic(s0, f, cnt);
      tracing_ = false;
    }
    join_dynamic_streams(s0);  // every queue stream back into the origin
  }
  for (size_t i = 1; i < slots_.size(); ++i) {
    hs_ok(hs_event_record(slots_[i].t_end, slots_[i].origin), "end record");
    hs_ok(hs_stream_wait(s0.origin, slots_[i].t_end), "end wait");
  }
  hs_ok(hs_event_record(s0.t_end, s0.origin), "end record");
  hs_ok(hs_event_sync(s0.t_end), "end sync");
  if (elapsed_ns) hs_ok(hs_event_elapsed_ns(s0.t_start, s0.t_end, elapsed_ns), "elapsed");
  ++runs_;
  batches_run_ += nb;
}

std::string Engine::info(const std::string& what) const {
  using json::Value;
  Value out = Value::make_object();
  auto pairs = [](const auto& v, auto a, auto b) {
    Value arr = Value::make_array();
    for (const auto& x : v) {
      Value p = Value::make_array();
      p.push_back(Value::of(static_cast<long long>(x.*a)));
      p.push_back(Value::of(static_cast<long long>(x.*b)));
      arr.push_back(std::move(p));
    }
    return arr;
  };
  if (what == "plan") {
    out.set("mode", Value::of(std::string(cfg_.graph_mode ? "graph" : "dynamic")));
    out.set("batch", Value::of(static_cast<long long>(cfg_.batch)));
    out.set("slots", Value::of(static_cast<long long>(cfg_.slots)));
    out.set("kernels", Value::of(static_cast<long long>(g_.kernels.size())));
    out.set("edges", Value::of(static_cast<long long>(g_.edges.size())));
    out.set("components", Value::of(static_cast<long long>(sched_->components().size())));
    // graph mode: the captured plan; dynamic mode: what Alg. 1 dispatched in the
    // last batch of the last run (timing-dependent for eager / HEFT)
    const bool dyn = !cfg_.graph_mode;
    out.set("dispatches", pairs(dyn ? last_dispatches_ : plan_.dispatches, &DispatchRecord::component,
                                &DispatchRecord::device));
    out.set("dispatches_source", Value::of(std::string(dyn ? "last dynamic run" : "captured plan")));
    long long streams = 0;
    for (const auto& sl : slots_) streams += static_cast<long long>(sl.streams.size());
    out.set("streams", Value::of(streams));
    out.set("device_bytes", Value::of(static_cast<long long>(device_bytes_)));
    // liveness planner: bytes per instance per slot of the pooled (arena) buffers,
    // against one allocation per output buffer
    out.set("arena_bytes_per_instance", Value::of(static_cast<long long>(pooled_bytes_per_instance_)));
    out.set("all_outputs_bytes_per_instance", Value::of(static_cast<long long>(unpooled_bytes_per_instance_)));
    long long resident_groups = 0;
    for (const auto& gr : groups_) resident_groups += gr.resident ? 1 : 0;
    out.set("resident_groups", Value::of(resident_groups));
    out.set("instance_groups", Value::of(static_cast<long long>(groups_.size()) - resident_groups));
    out.set("memory_domains", Value::of(static_cast<long long>(dctx_.size())));
    Value gpus = Value::make_array();
    for (int gpu : dom_gpu_) gpus.push_back(Value::of(static_cast<long long>(gpu)));
    out.set("domain_gpus", std::move(gpus));
    out.set("peer_copies_per_batch", Value::of(static_cast<long long>(peer_in_.size())));
    out.set("captured", Value::of(static_cast<long long>(capture_ok_ && cfg_.graph_mode ? 1 : 0)));
    out.set("ramp_batch", Value::of(static_cast<long long>(ramp_)));
    out.set("dynamic_fused", Value::of(static_cast<long long>(dyn_fused_ ? 1 : 0)));
    out.set("aliased_inputs", Value::of(static_cast<long long>(alias_.size())));
    out.set("grouped_launches", Value::of(static_cast<long long>(fuse_groups_.size())));
    Value rw = Value::make_object();
    for (const auto& [rule, n] : rewrites_) rw.set(rule, Value::of(static_cast<long long>(n)));
    out.set("chain_rewrites", std::move(rw));
    out.set("launches_per_batch", Value::of(static_cast<long long>(launches_per_batch_)));
  } else if (what == "stats") {
    out.set("launches_per_batch", Value::of(static_cast<long long>(launches_per_batch_)));
    // dynamic mode host cost: time in dispatch (setup of streams/events + launches)
    // and waiting for completion callbacks, summed over all runs
    out.set("host_dispatches", Value::of(static_cast<long long>(host_dispatches_)));
    out.set("host_dispatch_us", Value::real(double(host_dispatch_ns_) / 1e3));
    out.set("host_wait_us", Value::real(double(host_wait_ns_) / 1e3));
    out.set("runs", Value::of(static_cast<long long>(runs_)));
    out.set("batches", Value::of(static_cast<long long>(batches_run_)));
    // last whole-run graph capture: input groups / outputs used in place (zero copy)
    out.set("zero_copy_groups", Value::of(static_cast<long long>(zero_copy_groups_)));
    out.set("zero_copy_outputs", Value::of(static_cast<long long>(zero_copy_outputs_)));
  } else if (what == "trace") {
    // SPEC.md:435 trace records of the first batch of the last run (times in ms
    // from the run's start event): event id = position in issue order.
    static const char* kinds[3] = {"write", "ndrange", "read"};
    Value arr = Value::make_array();
    long long id = 0;
    for (const auto& r : trace_) {
      int64_t a = 0, b = 0;
      hs_ok(hs_event_elapsed_ns(slots_.front().t_start, r.t0, &a), "trace elapsed");
      hs_ok(hs_event_elapsed_ns(slots_.front().t_start, r.t1, &b), "trace elapsed");
      Value rec = Value::make_object();
      rec.set("event", Value::of(id++));
      rec.set("kind", Value::of(std::string(kinds[r.kind])));
      rec.set("label", Value::of(r.label));
      rec.set("kernel", Value::of(static_cast<long long>(r.kernel)));
      rec.set("component", Value::of(static_cast<long long>(r.component)));
      rec.set("device", Value::of(static_cast<long long>(r.device)));
      rec.set("queue", Value::of(static_cast<long long>(r.queue)));
      rec.set("channel", Value::of(-1LL));
      rec.set("start", Value::real(double(a) / 1e6));
      rec.set("finish", Value::real(double(b) / 1e6));
      arr.push_back(std::move(rec));
    }
    out.set("trace", std::move(arr));
    out.set("dispatches", pairs(trace_dispatch_, &DispatchRecord::component, &DispatchRecord::device));
    out.set("mode", Value::of(std::string(cfg_.graph_mode ? "graph" : "dynamic")));
    out.set("batch", Value::of(static_cast<long long>(cfg_.batch)));
  } else if (what == "completions") {
    out.set("completions", pairs(last_log_, &Completion::component, &Completion::event));
    out.set("dispatches", pairs(last_dispatches_, &DispatchRecord::component, &DispatchRecord::device));
  } else {
    fail(Errc::invalid_param, "unknown info '" + what + "'");
  }
  return json::dump(out, -1);
}

}  // namespace hetsim

// ------------------------------------------------------------------ C ABI
namespace {

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return HS_OK;
  } catch (const hetsim::Error& e) {
    const int status = hetsim::exit_code_for(e.code()) == 2 ? HS_ERR_INVALID
                       : e.code() == hetsim::Errc::device_error ? HS_ERR_CUDA
                                                                : HS_ERR_RUNTIME;
    return hs__set_error(status, static_cast<int>(e.code()), e.what());
  } catch (const std::exception& e) {
    return hs__set_error(HS_ERR_RUNTIME, -1, e.what());
  }
}

}  // namespace

extern "C" {

int hs_engine_create(const char* config_json, hs_engine_t* out) {
  return guarded([&] {
    using namespace hetsim;
    if (!out) fail(Errc::invalid_param, "null out");
    json::Value c;
    try {
      c = json::parse(config_json ? config_json : "");
    } catch (const std::exception& e) {
      fail(Errc::malformed_spec, std::string("engine config: ") + e.what());
    }
    EngineConfig cfg;
    cfg.spec_text = c.at("spec").as_string();
    if (const json::Value* p = c.find("params"))
      for (const auto& [k, v] : p->object_items()) cfg.params[k] = v.as_int64();
    if (const json::Value* v = c.find("gpu")) cfg.gpu = v->as_int();
    if (const json::Value* v = c.find("policy")) cfg.policy = policy_from_name(v->as_string());
    if (const json::Value* v = c.find("mode")) {
      if (v->as_string() != "graph" && v->as_string() != "dynamic") fail(Errc::invalid_param, "mode must be graph|dynamic");
      cfg.graph_mode = v->as_string() == "graph";
    }
    if (const json::Value* v = c.find("batch")) cfg.batch = v->as_int();
    if (const json::Value* v = c.find("slots")) cfg.slots = v->as_int();
    if (const json::Value* v = c.find("math")) {
      const std::string m = v->as_string();
      if (m == "tf32x3") cfg.math = HS_MATH_TF32X3;
      else if (m == "tf32") cfg.math = HS_MATH_TF32;
      else if (m == "simt") cfg.math = HS_MATH_FP32_SIMT;
      else if (m == "bf16x3") cfg.math = HS_MATH_BF16X3;
      else fail(Errc::invalid_param, "math must be tf32x3|tf32|bf16x3|simt");
    }
    if (const json::Value* v = c.find("trace")) cfg.trace = v->as_int() != 0;
    if (const json::Value* v = c.find("cpu_devices"))
      for (const json::Value* x : v->items()) cfg.cpu_devices.insert(x->as_int());
    if (const json::Value* v = c.find("device_gpus"))
      for (const auto& [k, g] : v->object_items()) cfg.device_gpus[std::stoi(k)] = g.as_int();
    if (const json::Value* v = c.find("domain_per_device")) cfg.domain_per_device = v->as_int() != 0;
    if (const json::Value* v = c.find("ramp")) {
      cfg.ramp = int(v->as_int());
      if (cfg.ramp < 0) fail(Errc::invalid_param, "ramp must be >= 0");
    }
    if (const json::Value* v = c.find("dynamic_fuse")) cfg.dynamic_fuse = v->as_int() != 0;
    if (const json::Value* v = c.find("deterministic")) cfg.deterministic = v->as_int() != 0;
    if (const json::Value* v = c.find("liveness")) cfg.liveness = v->as_int() != 0;
    if (const json::Value* v = c.find("run_graph")) cfg.run_graph = v->as_int() != 0;
    if (const json::Value* v = c.find("zero_copy")) cfg.zero_copy = v->as_int() != 0;
    if (const json::Value* v = c.find("fuse")) {
      cfg.fuse = v->as_int();
      if (cfg.fuse < 0 || cfg.fuse > 3) fail(Errc::invalid_param, "fuse must be 0, 1, 2 or 3");
    }
    *out = reinterpret_cast<hs_engine_t>(new Engine(std::move(cfg)));
  });
}

int hs_engine_destroy(hs_engine_t e) {
  return guarded([&] { delete reinterpret_cast<hetsim::Engine*>(e); });
}

int hs_engine_bind(hs_engine_t e, int kernel, int pos, void* ptr, int64_t stride_bytes, int64_t count,
                   int on_device) {
  return guarded([&] {
    if (!e) hetsim::fail(hetsim::Errc::invalid_param, "null engine");
    reinterpret_cast<hetsim::Engine*>(e)->bind(kernel, pos, ptr, stride_bytes, count, on_device != 0);
  });
}

int hs_engine_run(hs_engine_t e, int64_t first, int64_t n, int64_t* elapsed_ns) {
  return guarded([&] {
    if (!e) hetsim::fail(hetsim::Errc::invalid_param, "null engine");
    reinterpret_cast<hetsim::Engine*>(e)->run(first, n, elapsed_ns);
  });
}

int hs_engine_info(hs_engine_t e, const char* what, char** out_json) {
  return guarded([&] {
    if (!e || !what || !out_json) hetsim::fail(hetsim::Errc::invalid_param, "null argument");
    std::string s = reinterpret_cast<hetsim::Engine*>(e)->info(what);
    char* buf = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(buf, s.c_str(), s.size() + 1);
    *out_json = buf;
  });
}

}  // extern "C"
