// DAG specification: parse / validate / serialize.
//
// Validation order and error codes restate proj/src/spec_model.cpp:211-343
// so that invalid documents fail with the same Errc as the reference:
//   kernels (ids, names, dev, workDimension, globalWorkSize, buffers,
//   varArguments, src, dense arg positions, duplicate ids) -> depends -> tc
//   -> cq -> edge endpoint checks -> acyclicity -> tc partition checks.
// serialize() emits the reference's key order and pretty-print format
// (proj/src/spec_model.cpp:353-386) through our own JSON printer.
#include "hetsim/spec_model.hpp"

#include <algorithm>
#include <limits>

#include "hetsim/errors.hpp"
#include "json.hpp"

namespace hetsim {

using json::Value;

int elem_width(ElemType t) { return (t == ElemType::f64 || t == ElemType::i64) ? 8 : 4; }

const char* elem_type_name(ElemType t) {
  switch (t) {
    case ElemType::f32: return "float32";
    case ElemType::i32: return "int32";
    case ElemType::f64: return "float64";
    case ElemType::i64: return "int64";
  }
  return "float32";
}

const char* device_type_name(DeviceType t) { return t == DeviceType::cpu ? "cpu" : "gpu"; }

// ---------------------------------------------------------------------------
// KernelSpec / DagSpec accessors
// ---------------------------------------------------------------------------

namespace {

std::vector<const BufferSpec*> merged_by_pos(const std::vector<BufferSpec>& a, const std::vector<BufferSpec>& b) {
  std::vector<const BufferSpec*> out;
  out.reserve(a.size() + b.size());
  for (const auto& x : a) out.push_back(&x);
  for (const auto& x : b) out.push_back(&x);
  std::stable_sort(out.begin(), out.end(), [](const BufferSpec* l, const BufferSpec* r) { return l->pos < r->pos; });
  return out;
}

}  // namespace

std::vector<const BufferSpec*> KernelSpec::input_side() const { return merged_by_pos(input_buffers, io_buffers); }
std::vector<const BufferSpec*> KernelSpec::output_side() const { return merged_by_pos(output_buffers, io_buffers); }

const BufferSpec* KernelSpec::buffer_at(int pos) const {
  for (const auto* list : {&input_buffers, &output_buffers, &io_buffers})
    for (const auto& b : *list)
      if (b.pos == pos) return &b;
  return nullptr;
}

const VarArg* KernelSpec::var_arg_at(int pos) const {
  for (const auto& v : var_args)
    if (v.pos == pos) return &v;
  return nullptr;
}

int DagSpec::index_of(int id) const {
  if (index_size_ != kernels.size()) {
    index_.clear();
    index_.reserve(kernels.size() * 2);
    for (size_t i = 0; i < kernels.size(); ++i) index_.emplace(kernels[i].id, int(i));  // first wins
    index_size_ = kernels.size();
  }
  auto it = index_.find(id);
  if (it != index_.end() && size_t(it->second) < kernels.size() && kernels[it->second].id == id) return it->second;
  // Stale index (kernels edited in place): fall back to a scan and rebuild next time.
  for (size_t i = 0; i < kernels.size(); ++i) {
    if (kernels[i].id == id) {
      index_size_ = static_cast<size_t>(-1);
      return int(i);
    }
  }
  return -1;
}

const KernelSpec& DagSpec::kernel(int id) const {
  int i = index_of(id);
  if (i < 0) fail(Errc::unknown_kernel_ref, "no kernel with id " + std::to_string(id));
  return kernels[size_t(i)];
}

bool DagSpec::has_kernel(int id) const { return index_of(id) >= 0; }

std::map<int, std::set<int>> DagSpec::kernel_successors() const {
  std::map<int, std::set<int>> out;
  for (const auto& k : kernels) out[k.id];
  for (const auto& e : edges) out[e.src_kernel].insert(e.dst_kernel);
  return out;
}

std::map<int, std::set<int>> DagSpec::kernel_predecessors() const {
  std::map<int, std::set<int>> out;
  for (const auto& k : kernels) out[k.id];
  for (const auto& e : edges) out[e.dst_kernel].insert(e.src_kernel);
  return out;
}

std::map<std::pair<int, int>, int> DagSpec::producer_edge() const {
  std::map<std::pair<int, int>, int> out;
  for (size_t i = 0; i < edges.size(); ++i) out[{edges[i].dst_kernel, edges[i].dst_pos}] = int(i);
  return out;
}

std::map<std::pair<int, int>, std::vector<int>> DagSpec::consumer_edges() const {
  std::map<std::pair<int, int>, std::vector<int>> out;
  for (size_t i = 0; i < edges.size(); ++i) out[{edges[i].src_kernel, edges[i].src_pos}].push_back(int(i));
  return out;
}

std::vector<int> DagSpec::topo_order() const {
  // Kahn's algorithm; the frontier is an ordered set so that the smallest
  // ready id is always taken first (deterministic, matches the reference).
  auto succ = kernel_successors();
  std::map<int, int> indeg;
  for (const auto& k : kernels) indeg[k.id] = 0;
  for (const auto& [src, dsts] : succ)
    for (int d : dsts) ++indeg[d];
  std::set<int> ready;
  for (const auto& [id, d] : indeg)
    if (d == 0) ready.insert(id);
  std::vector<int> order;
  order.reserve(kernels.size());
  while (!ready.empty()) {
    int id = *ready.begin();
    ready.erase(ready.begin());
    order.push_back(id);
    for (int d : succ[id])
      if (--indeg[d] == 0) ready.insert(d);
  }
  if (order.size() != kernels.size()) fail(Errc::cycle_detected, "the depends edges form a cycle");
  return order;
}

std::map<int, int> DagSpec::component_of() const {
  std::map<int, int> out;
  for (size_t c = 0; c < tc.size(); ++c)
    for (int id : tc[c]) out[id] = int(c);
  return out;
}

// ---------------------------------------------------------------------------
// parse_spec
// ---------------------------------------------------------------------------

namespace {

ElemType elem_type_from(const std::string& s) {
  if (s == "float32") return ElemType::f32;
  if (s == "int32") return ElemType::i32;
  if (s == "float64") return ElemType::f64;
  if (s == "int64") return ElemType::i64;
  fail(Errc::malformed_spec, "buffer type '" + s + "' is not one of the element types");
}

DeviceType device_type_from(const std::string& s) {
  if (s == "cpu") return DeviceType::cpu;
  if (s == "gpu") return DeviceType::gpu;
  fail(Errc::malformed_spec, "dev '" + s + "' is neither gpu nor cpu");
}

// A symbolic field may be written as a JSON string or as an integer.
std::string symbolic(const Value& v) {
  std::string s = v.is_string() ? v.as_string() : std::to_string(v.as_int64());
  validate_expr(s);
  return s;
}

BufferSpec read_buffer(const Value& j, int kernel_id, BufferKind kind) {
  if (!j.is_object()) fail(Errc::malformed_spec, "each buffer is a JSON object");
  if (!j.contains("type") || !j.contains("size") || !j.contains("pos"))
    fail(Errc::malformed_spec, "a buffer lacks one of type, size, pos");
  BufferSpec b;
  b.kernel = kernel_id;
  b.kind = kind;
  b.type = elem_type_from(j.at("type").as_string());
  b.size_expr = symbolic(j.at("size"));
  b.pos = j.at("pos").as_int();
  if (b.pos < 0) fail(Errc::malformed_spec, "negative buffer position");
  return b;
}

// Every argument slot 0..max(pos) is taken by exactly one buffer or var-arg.
void check_positions(const KernelSpec& k) {
  std::map<int, int> used;
  auto take = [&](int pos, const char* what) {
    if (pos < 0) fail(Errc::malformed_spec, "negative position in " + std::string(what));
    if (++used[pos] > 1)
      fail(Errc::arg_position_clash, "two arguments of kernel " + std::to_string(k.id) + " share position " + std::to_string(pos));
  };
  for (const auto& b : k.input_buffers) take(b.pos, "a buffer");
  for (const auto& b : k.output_buffers) take(b.pos, "a buffer");
  for (const auto& b : k.io_buffers) take(b.pos, "a buffer");
  for (const auto& v : k.var_args) take(v.pos, "a varArgument");
  if (used.empty()) return;
  int hi = used.rbegin()->first;
  if (int(used.size()) != hi + 1) {
    for (int p = 0; p <= hi; ++p)
      if (!used.count(p))
        fail(Errc::malformed_spec,
             "kernel " + std::to_string(k.id) + " has a gap at argument position " + std::to_string(p));
  }
}

// Member `key` of `root`, or an empty array. Returned by reference so that
// range-for over `.items()` never points into a destroyed temporary.
const Value& list_or_empty(const Value& root, const char* key) {
  static const Value kEmpty = Value::make_array();
  const Value* v = root.find(key);
  return v ? *v : kEmpty;
}

void read_document(const Value& root, DagSpec& g) {
  for (const Value* pk : root.at("kernels").items()) {
    const Value& jk = *pk;
    KernelSpec k;
    k.id = jk.at("id").as_int();
    if (k.id < 0) fail(Errc::malformed_spec, "negative kernel id");
    k.name = jk.at("name").as_string();
    k.dev = device_type_from(jk.at("dev").as_string());
    if (!jk.is_object()) throw json::TypeError("kernel entry must be an object");
    const Value* wd = jk.find("workDimension");
    k.work_dimension = wd ? wd->as_int() : 1;
    if (k.work_dimension < 1 || k.work_dimension > 3) fail(Errc::malformed_spec, "workDimension outside 1..3");
    if (const Value* gws = jk.find("globalWorkSize")) {
      if (!gws->is_array() || gws->size() != 3) fail(Errc::malformed_spec, "globalWorkSize is not a list of three");
      for (int i = 0; i < 3; ++i) k.global_work_size[size_t(i)] = symbolic((*gws)[size_t(i)]);
    }
    for (const Value* jb : list_or_empty(jk, "inputBuffers").items())
      k.input_buffers.push_back(read_buffer(*jb, k.id, BufferKind::input));
    for (const Value* jb : list_or_empty(jk, "outputBuffers").items())
      k.output_buffers.push_back(read_buffer(*jb, k.id, BufferKind::output));
    for (const Value* jb : list_or_empty(jk, "ioBuffers").items())
      k.io_buffers.push_back(read_buffer(*jb, k.id, BufferKind::io));
    for (const Value* jv : list_or_empty(jk, "varArguments").items()) {
      VarArg v;
      v.type = jv->at("type").as_string();
      v.pos = jv->at("pos").as_int();
      v.value = symbolic(jv->at("value"));
      k.var_args.push_back(std::move(v));
    }
    const Value* src = jk.find("src");
    k.src_path = src ? src->as_string() : std::string();
    check_positions(k);
    if (g.has_kernel(k.id)) fail(Errc::malformed_spec, "kernel id " + std::to_string(k.id) + " is used twice");
    g.kernels.push_back(std::move(k));
  }

  for (const Value* je : list_or_empty(root, "depends").items()) {
    if (!je->is_array() || je->size() != 4) fail(Errc::malformed_spec, "a depends entry is not [src, src_pos, dst, dst_pos]");
    g.edges.push_back(DagEdge{(*je)[0].as_int(), (*je)[1].as_int(), (*je)[2].as_int(), (*je)[3].as_int()});
  }

  for (const Value* jt : list_or_empty(root, "tc").items()) {
    std::vector<int> comp;
    for (const Value* id : jt->items()) comp.push_back(id->as_int());
    g.tc.push_back(std::move(comp));
  }

  for (const Value* jc : list_or_empty(root, "cq").items()) {
    int dev = jc->at("device").as_int();
    int n = jc->at("queues").as_int();
    if (n < 0) fail(Errc::malformed_spec, "negative queue count in cq");
    g.cq[dev] = n;
  }
}

}  // namespace

DagSpec parse_spec(const std::string& text, const ParamMap& params) {
  Value root;
  try {
    root = json::parse(text);
  } catch (const json::ParseError& e) {
    fail(Errc::malformed_spec, e.what());
  }
  if (!root.is_object() || !root.contains("kernels"))
    fail(Errc::malformed_spec, "the document is not an object with a kernels list");

  DagSpec g;
  g.params = params;
  try {
    read_document(root, g);
  } catch (const json::TypeError& e) {
    fail(Errc::malformed_spec, e.what());
  }

  // Edges: known endpoints, output-side source, input-side target, one producer per input.
  std::set<std::pair<int, int>> fed;
  for (const auto& e : g.edges) {
    if (!g.has_kernel(e.src_kernel)) fail(Errc::unknown_kernel_ref, "depends edge from missing kernel " + std::to_string(e.src_kernel));
    if (!g.has_kernel(e.dst_kernel)) fail(Errc::unknown_kernel_ref, "depends edge into missing kernel " + std::to_string(e.dst_kernel));
    const BufferSpec* s = g.kernel(e.src_kernel).buffer_at(e.src_pos);
    if (!s || s->kind == BufferKind::input)
      fail(Errc::malformed_spec, "edge source (" + std::to_string(e.src_kernel) + "," + std::to_string(e.src_pos) +
                                     ") does not produce data (input buffer or no buffer)");
    const BufferSpec* d = g.kernel(e.dst_kernel).buffer_at(e.dst_pos);
    if (!d || d->kind == BufferKind::output)
      fail(Errc::malformed_spec, "edge target (" + std::to_string(e.dst_kernel) + "," + std::to_string(e.dst_pos) +
                                     ") does not consume data (output buffer or no buffer)");
    if (!fed.insert({e.dst_kernel, e.dst_pos}).second)
      fail(Errc::malformed_spec, "input buffer (" + std::to_string(e.dst_kernel) + "," + std::to_string(e.dst_pos) +
                                     ") is fed by more than one edge");
  }

  g.topo_order();  // CycleDetected

  // tc: non-empty parts, known ids, disjoint, one device type per part, covering.
  std::set<int> seen;
  for (const auto& comp : g.tc) {
    if (comp.empty()) fail(Errc::partition_error, "a tc entry lists no kernels");
    const KernelSpec* first = nullptr;
    for (int id : comp) {
      if (!g.has_kernel(id)) fail(Errc::partition_error, "tc names missing kernel " + std::to_string(id));
      if (!seen.insert(id).second) fail(Errc::partition_error, "tc lists kernel " + std::to_string(id) + " more than once");
      const KernelSpec& k = g.kernel(id);
      if (!first) first = &k;
      else if (k.dev != first->dev) fail(Errc::partition_error, "a tc entry mixes gpu and cpu kernels");
    }
  }
  if (seen.size() != g.kernels.size()) fail(Errc::partition_error, "some kernel belongs to no tc entry");
  return g;
}

// ---------------------------------------------------------------------------
// serialize / buffer_bytes
// ---------------------------------------------------------------------------

namespace {

Value str(const std::string& s) { return Value::of(s); }
Value num(long long i) { return Value::of(i); }

Value buffer_value(const BufferSpec& b) {
  Value o = Value::make_object();
  o.set("type", str(elem_type_name(b.type)));
  o.set("size", str(b.size_expr));
  o.set("pos", num(b.pos));
  return o;
}

Value buffer_list(const std::vector<BufferSpec>& v) {
  Value a = Value::make_array();
  for (const auto& b : v) a.push_back(buffer_value(b));
  return a;
}

}  // namespace

json::Value spec_to_json(const DagSpec& g) {
  Value root = Value::make_object();
  Value kernels = Value::make_array();
  for (const auto& k : g.kernels) {
    Value jk = Value::make_object();
    jk.set("id", num(k.id));
    jk.set("name", str(k.name));
    jk.set("dev", str(device_type_name(k.dev)));
    jk.set("workDimension", num(k.work_dimension));
    Value gws = Value::make_array();
    for (const auto& s : k.global_work_size) gws.push_back(str(s));
    jk.set("globalWorkSize", std::move(gws));
    jk.set("inputBuffers", buffer_list(k.input_buffers));
    jk.set("outputBuffers", buffer_list(k.output_buffers));
    jk.set("ioBuffers", buffer_list(k.io_buffers));
    Value va = Value::make_array();
    for (const auto& v : k.var_args) {
      Value o = Value::make_object();
      o.set("type", str(v.type));
      o.set("pos", num(v.pos));
      o.set("value", str(v.value));
      va.push_back(std::move(o));
    }
    jk.set("varArguments", std::move(va));
    jk.set("src", str(k.src_path));
    kernels.push_back(std::move(jk));
  }
  root.set("kernels", std::move(kernels));
  Value tc = Value::make_array();
  for (const auto& comp : g.tc) {
    Value c = Value::make_array();
    for (int id : comp) c.push_back(num(id));
    tc.push_back(std::move(c));
  }
  root.set("tc", std::move(tc));
  Value cq = Value::make_array();
  for (const auto& [dev, n] : g.cq) {
    Value o = Value::make_object();
    o.set("device", num(dev));
    o.set("queues", num(n));
    cq.push_back(std::move(o));
  }
  root.set("cq", std::move(cq));
  Value deps = Value::make_array();
  for (const auto& e : g.edges) {
    Value r = Value::make_array();
    r.push_back(num(e.src_kernel));
    r.push_back(num(e.src_pos));
    r.push_back(num(e.dst_kernel));
    r.push_back(num(e.dst_pos));
    deps.push_back(std::move(r));
  }
  root.set("depends", std::move(deps));
  return root;
}

std::string serialize(const DagSpec& g) { return json::dump(spec_to_json(g), 2) + "\n"; }

long long buffer_bytes(const BufferSpec& b, const ParamMap& params) {
  __int128 bytes = __int128(eval_positive(b.size_expr, params)) * elem_width(b.type);
  if (bytes > std::numeric_limits<long long>::max()) fail(Errc::numeric_overflow, "buffer size in bytes overflows 64 bits");
  return static_cast<long long>(bytes);
}

}  // namespace hetsim
