// Command-queue construction (Alg. 1 setup_cq / enq / set_dependencies /
// set_callbacks). Rules, with their sources:
//
//  enq(k,q)          SPEC.md:219-227, cq_builder.hpp:54-58
//    [dependent writes: k in FRONT(T), one per inter in-edge, ascending pos]
//    [isolated writes, ascending pos] [ndrange]
//    [isolated reads, ascending pos]
//    [dependent reads: k in END(T), one per inter out-edge, ascending pos then edge index]
//  set_dependencies  SPEC.md:229-236, PAPER.md:193 — cross-queue pairs only:
//    (i) write->ndrange, (ii) ndrange->read, (iii) ndrange->ndrange across an intra edge
//  set_callbacks     SPEC.md:248-255, PAPER.md:301-304 — GPU: dependent reads of END
//    kernels; CPU: ndrange of END kernels; plus the terminal command of every queue
//  setup_cq          cq_builder.hpp:72-76, SPEC.md:238-246 — kernels in component
//    topological order (ascending-id ties), queue = position mod r, then an
//    acyclicity check of in-queue order + E_Q.
#include "hetsim/cq_builder.hpp"

#include <algorithm>
#include <map>

#include "hetsim/errors.hpp"
#include "../core/json.hpp"

namespace hetsim {

const char* cmd_kind_name(CmdKind k) {
  switch (k) {
    case CmdKind::write: return "write";
    case CmdKind::ndrange: return "ndrange";
    case CmdKind::read: return "read";
  }
  return "?";
}

const Command& CommandQueueStructure::command_of(int event) const {
  if (event < 0 || size_t(event) >= event_pos.size()) fail(Errc::unknown_event, "event " + std::to_string(event));
  auto [q, i] = event_pos[size_t(event)];
  return queues[size_t(q)][size_t(i)];
}

std::optional<int> CommandQueueStructure::ndrange_event(int kernel) const {
  for (const auto& q : queues)
    for (const auto& c : q)
      if (c.kind == CmdKind::ndrange && c.kernel == kernel) return c.event;
  return std::nullopt;
}

std::vector<int> CommandQueueStructure::terminal_events() const {
  std::vector<int> out;
  for (const auto& q : queues)
    if (!q.empty()) out.push_back(q.back().event);
  return out;
}

namespace {

int count_kind(const CommandQueueStructure& cqs, CmdKind k) {
  int n = 0;
  for (const auto& q : cqs.queues)
    for (const auto& c : q) n += (c.kind == k);
  return n;
}

void push(CommandQueueStructure& cqs, int q, Command c, int (&counters)[3]) {
  static const char kPrefix[3] = {'w', 'e', 'r'};
  int kind = static_cast<int>(c.kind);
  c.event = cqs.event_count++;
  c.label = std::string(1, kPrefix[kind]) + std::to_string(++counters[kind]);
  cqs.event_pos.emplace_back(q, int(cqs.queues[size_t(q)].size()));
  cqs.queues[size_t(q)].push_back(std::move(c));
}

Command transfer(CmdKind kind, const KernelSpec& k, const BufferSpec& b, bool dependent, int edge,
                 const DagSpec& g) {
  Command c;
  c.kind = kind;
  c.kernel = k.id;
  c.buffer = BufferRef{k.id, b.pos};
  c.dependent = dependent;
  c.bytes = buffer_bytes(b, g.params);
  c.edge = edge;
  return c;
}

}  // namespace

void enq(int kernel, int q, const TaskComponent& t, const DagSpec& g, const EdgeClasses& ec,
         CommandQueueStructure& cqs) {
  if (cqs.processed.count(kernel)) fail(Errc::already_processed, "kernel " + std::to_string(kernel));
  if (q < 0 || size_t(q) >= cqs.queues.size())
    fail(Errc::invalid_param, "queue index " + std::to_string(q) + " out of range");
  const KernelSpec& k = g.kernel(kernel);
  // Per-kind label counters continue from what the structure already holds.
  int counters[3] = {count_kind(cqs, CmdKind::write), count_kind(cqs, CmdKind::ndrange),
                     count_kind(cqs, CmdKind::read)};
  const auto ins = k.input_side();
  const auto outs = k.output_side();

  if (t.front.count(kernel)) {
    for (const BufferSpec* b : ins)
      for (size_t e = 0; e < g.edges.size(); ++e)
        if (g.edges[e].dst_kernel == kernel && g.edges[e].dst_pos == b->pos && ec.edge_kind[e] == EdgeKind::inter)
          push(cqs, q, transfer(CmdKind::write, k, *b, true, int(e), g), counters);
  }
  for (const BufferSpec* b : ins)
    if (ec.write_class.at({kernel, b->pos}) == CopyClass::isolated)
      push(cqs, q, transfer(CmdKind::write, k, *b, false, -1, g), counters);

  Command nd;
  nd.kind = CmdKind::ndrange;
  nd.kernel = kernel;
  push(cqs, q, std::move(nd), counters);

  for (const BufferSpec* b : outs)
    if (ec.read_class.at({kernel, b->pos}) == CopyClass::isolated)
      push(cqs, q, transfer(CmdKind::read, k, *b, false, -1, g), counters);
  if (t.end.count(kernel)) {
    for (const BufferSpec* b : outs)
      for (size_t e = 0; e < g.edges.size(); ++e)
        if (g.edges[e].src_kernel == kernel && g.edges[e].src_pos == b->pos && ec.edge_kind[e] == EdgeKind::inter)
          push(cqs, q, transfer(CmdKind::read, k, *b, true, int(e), g), counters);
  }
  cqs.processed.insert(kernel);
}

void set_dependencies(int kernel, CommandQueueStructure& cqs, const TaskComponent& t, const DagSpec& g,
                      const EdgeClasses& ec) {
  (void)t;
  auto nd = cqs.ndrange_event(kernel);
  if (!nd) return;
  const int nd_q = cqs.event_pos[size_t(*nd)].first;
  auto add = [&](int from, int to) {
    if (cqs.event_pos[size_t(from)].first != cqs.event_pos[size_t(to)].first) cqs.deps.insert({from, to});
  };
  // (i) writes -> ndrange and (ii) ndrange -> reads of the same kernel.
  for (const auto& q : cqs.queues)
    for (const auto& c : q) {
      if (c.kernel != kernel) continue;
      if (c.kind == CmdKind::write) add(c.event, *nd);
      if (c.kind == CmdKind::read) add(*nd, c.event);
    }
  // (iii) ndrange -> ndrange across intra edges whose other end is already enqueued.
  for (size_t e = 0; e < g.edges.size(); ++e) {
    if (ec.edge_kind[e] != EdgeKind::intra) continue;
    const DagEdge& de = g.edges[e];
    if (de.dst_kernel == kernel && de.src_kernel != kernel) {
      if (auto src = cqs.ndrange_event(de.src_kernel)) add(*src, *nd);
    } else if (de.src_kernel == kernel && de.dst_kernel != kernel) {
      if (auto dst = cqs.ndrange_event(de.dst_kernel)) add(*nd, *dst);
    }
  }
  (void)nd_q;
}

void set_callbacks(const TaskComponent& t, DeviceType device_type, CommandQueueStructure& cqs, const DagSpec& g,
                   const EdgeClasses& ec) {
  (void)g;
  (void)ec;
  for (const auto& q : cqs.queues)
    for (const auto& c : q) {
      if (!t.end.count(c.kernel)) continue;
      bool mark = device_type == DeviceType::gpu ? (c.kind == CmdKind::read && c.dependent)
                                                 : (c.kind == CmdKind::ndrange);
      if (mark) {
        cqs.end_marks.insert(c.event);
        cqs.callbacks.insert(c.event);
      }
    }
  for (int ev : cqs.terminal_events()) cqs.callbacks.insert(ev);
}

namespace {

// Kahn order of the component's induced kernel subgraph, smallest id first.
std::vector<int> component_order(const TaskComponent& t, const DagSpec& g) {
  std::set<int> members(t.kernel_ids.begin(), t.kernel_ids.end());
  std::map<int, std::set<int>> succ;
  std::map<int, int> indeg;
  for (int k : t.kernel_ids) indeg[k] = 0;
  for (const auto& e : g.edges)
    if (members.count(e.src_kernel) && members.count(e.dst_kernel) && e.src_kernel != e.dst_kernel)
      if (succ[e.src_kernel].insert(e.dst_kernel).second) ++indeg[e.dst_kernel];
  std::set<int> ready;
  for (auto [k, d] : indeg)
    if (d == 0) ready.insert(k);
  std::vector<int> order;
  while (!ready.empty()) {
    int k = *ready.begin();
    ready.erase(ready.begin());
    order.push_back(k);
    for (int s : succ[k])
      if (--indeg[s] == 0) ready.insert(s);
  }
  if (order.size() != members.size()) fail(Errc::cycle_detected, "component " + std::to_string(t.id) + " is cyclic");
  return order;
}

void check_acyclic(const CommandQueueStructure& cqs) {
  const int n = cqs.event_count;
  std::vector<std::vector<int>> out(static_cast<size_t>(n));
  std::vector<int> indeg(static_cast<size_t>(n), 0);
  for (const auto& q : cqs.queues)
    for (size_t i = 1; i < q.size(); ++i) {
      out[size_t(q[i - 1].event)].push_back(q[i].event);
      ++indeg[size_t(q[i].event)];
    }
  for (auto [a, b] : cqs.deps) {
    out[size_t(a)].push_back(b);
    ++indeg[size_t(b)];
  }
  std::vector<int> stack;
  for (int i = 0; i < n; ++i)
    if (!indeg[size_t(i)]) stack.push_back(i);
  int seen = 0;
  while (!stack.empty()) {
    int v = stack.back();
    stack.pop_back();
    ++seen;
    for (int w : out[size_t(v)])
      if (--indeg[size_t(w)] == 0) stack.push_back(w);
  }
  if (seen != n) fail(Errc::deadlock, "command structure of component " + std::to_string(cqs.component) + " is cyclic");
}

}  // namespace

CommandQueueStructure setup_cq(const TaskComponent& t, int device_id, DeviceType device_type, int r,
                               const DagSpec& g, const EdgeClasses& ec) {
  if (t.kernel_ids.empty()) fail(Errc::empty_component, "component " + std::to_string(t.id));
  if (r < 1) fail(Errc::invalid_param, "device " + std::to_string(device_id) + " needs at least one queue");
  CommandQueueStructure cqs;
  cqs.component = t.id;
  cqs.device = device_id;
  cqs.queues.resize(size_t(r));
  auto order = component_order(t, g);
  for (size_t i = 0; i < order.size(); ++i) {
    enq(order[i], int(i % size_t(r)), t, g, ec, cqs);
    set_dependencies(order[i], cqs, t, g, ec);
  }
  set_callbacks(t, device_type, cqs, g, ec);
  check_acyclic(cqs);
  return cqs;
}

std::string to_debug_json(const CommandQueueStructure& cqs) {
  using json::Value;
  auto label = [&](int ev) { return Value::of(cqs.command_of(ev).label); };
  Value root = Value::make_object();
  root.set("component", Value::of(cqs.component));
  root.set("device", Value::of(cqs.device));
  Value queues = Value::make_array();
  for (const auto& q : cqs.queues) {
    Value lq = Value::make_array();
    for (const auto& c : q) lq.push_back(Value::of(c.label));
    queues.push_back(std::move(lq));
  }
  root.set("queues", std::move(queues));
  Value deps = Value::make_array();
  for (auto [a, b] : cqs.deps) {
    Value p = Value::make_array();
    p.push_back(label(a));
    p.push_back(label(b));
    deps.push_back(std::move(p));
  }
  root.set("deps", std::move(deps));
  Value cb = Value::make_array();
  for (int ev : cqs.callbacks) cb.push_back(label(ev));
  root.set("callbacks", std::move(cb));
  Value em = Value::make_array();
  for (int ev : cqs.end_marks) em.push_back(label(ev));
  root.set("end_marks", std::move(em));
  Value cmds = Value::make_array();
  for (int ev = 0; ev < cqs.event_count; ++ev) {
    const Command& c = cqs.command_of(ev);
    Value o = Value::make_object();
    o.set("event", Value::of(c.event));
    o.set("label", Value::of(c.label));
    o.set("kind", Value::of(std::string(cmd_kind_name(c.kind))));
    o.set("kernel", Value::of(c.kernel));
    o.set("queue", Value::of(cqs.event_pos[size_t(ev)].first));
    if (c.buffer) {
      Value b = Value::make_array();
      b.push_back(Value::of(c.buffer->kernel));
      b.push_back(Value::of(c.buffer->pos));
      o.set("buffer", std::move(b));
      o.set("dependent", Value::of(static_cast<long long>(c.dependent)));
      o.set("bytes", Value::of(c.bytes));
      o.set("edge", Value::of(c.edge));
    }
    cmds.push_back(std::move(o));
  }
  root.set("commands", std::move(cmds));
  return json::dump(root, 2) + "\n";
}

}  // namespace hetsim
