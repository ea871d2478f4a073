// hs_query: JSON-in / JSON-out access to the host-side C++ API (spec model,
// analysis, command-queue construction, scheduling) through the C ABI.
//
// Used by the Python mirror (paper_2009_07482_b200/hetsim.py) and by the
// differential tests, which send the same request to the reference shim
// (oracle/ref_shim.cpp) for the operations the reference implements.
#include <cstdlib>
#include <cstring>
#include <string>

#include "../core/json.hpp"
#include "hetsim/cq_builder.hpp"
#include "hetsim/errors.hpp"
#include "hetsim/expr.hpp"
#include "hetsim/graph_analysis.hpp"
#include "hetsim/rational.hpp"
#include "hetsim/platform_sim.hpp"
#include "hetsim/scheduler.hpp"
#include "hetsim/spec_model.hpp"
#include "hetsim_c.h"

using namespace hetsim;
using json::Value;

namespace hetsim {
json::Value spec_to_json(const DagSpec& g);  // spec_model.cpp
}

namespace {

Value V(long long i) { return Value::of(i); }
Value S(const std::string& s) { return Value::of(s); }

Value ints(const std::vector<int>& v) {
  Value a = Value::make_array();
  for (int x : v) a.push_back(V(x));
  return a;
}
Value ints(const std::set<int>& v) {
  Value a = Value::make_array();
  for (int x : v) a.push_back(V(x));
  return a;
}
Value triple(int a, int b, const char* c) {
  Value t = Value::make_array();
  t.push_back(V(a));
  t.push_back(V(b));
  t.push_back(S(c));
  return t;
}

ParamMap params_of(const Value& req) {
  ParamMap p;
  if (const Value* ps = req.find("params"))
    for (const auto& [k, v] : ps->object_items()) p[k] = v.as_int64();
  return p;
}

Value analyze(const DagSpec& g) {
  Value out = Value::make_object();
  out.set("topo_order", ints(g.topo_order()));
  Value comps = Value::make_array();
  for (const auto& t : derive_components(g)) {
    Value c = Value::make_object();
    c.set("id", V(t.id));
    c.set("kernels", ints(t.kernel_ids));
    c.set("dev_pref", S(device_type_name(t.dev_pref)));
    c.set("front", ints(t.front));
    c.set("end", ints(t.end));
    c.set("interior", ints(t.interior));
    comps.push_back(std::move(c));
  }
  out.set("components", std::move(comps));
  auto ec = classify_edges(g);
  Value kinds = Value::make_array();
  for (auto k : ec.edge_kind) kinds.push_back(S(k == EdgeKind::intra ? "intra" : "inter"));
  out.set("edge_kind", std::move(kinds));
  Value wc = Value::make_array(), rc = Value::make_array();
  for (const auto& [key, cls] : ec.write_class)
    wc.push_back(triple(key.first, key.second, cls == CopyClass::isolated ? "isolated" : "dependent"));
  for (const auto& [key, cls] : ec.read_class)
    rc.push_back(triple(key.first, key.second, cls == CopyClass::isolated ? "isolated" : "dependent"));
  out.set("write_class", std::move(wc));
  out.set("read_class", std::move(rc));
  Value succ = Value::make_array();
  for (const auto& [k, s] : g.kernel_successors()) {
    Value p = Value::make_array();
    p.push_back(V(k));
    p.push_back(ints(s));
    succ.push_back(std::move(p));
  }
  out.set("successors", std::move(succ));
  Value co = Value::make_array();
  for (const auto& [k, c] : g.component_of()) {
    Value p = Value::make_array();
    p.push_back(V(k));
    p.push_back(V(c));
    co.push_back(std::move(p));
  }
  out.set("component_of", std::move(co));
  return out;
}

Profiles profiles_of(const Value& req) {
  Profiles prof;
  if (const Value* t = req.find("times")) {
    for (const auto& [dev, per] : t->object_items()) {
      DeviceType dt = dev == "cpu" ? DeviceType::cpu : DeviceType::gpu;
      for (const auto& [k, v] : per.object_items())
        prof.time[{std::stoi(k), dt}] = v.is_string() ? Ratio::parse(v.as_string()) : Ratio(v.as_int64());
    }
  }
  return prof;
}

Value schedule(const DagSpec& g, const Value& req) {
  std::set<int> cpu_ids;
  if (const Value* c = req.find("cpu_devices"))
    for (const Value* v : c->items()) cpu_ids.insert(v->as_int());
  Platform p = Platform::from_spec(g, cpu_ids);
  Policy pol = policy_from_name(req.find("policy") ? req.at("policy").as_string() : "clustering");
  Profiles prof = profiles_of(req);
  ScheduleResult r;
  if (const Value* log = req.find("replay")) {
    std::vector<Completion> entries;
    for (const Value* e : log->items()) entries.push_back({(*e)[0].as_int(), (*e)[1].as_int()});
    ReplayExecutor ex(std::move(entries));
    r = run_schedule(g, p, prof, pol, ex);
  } else {
    PlanExecutor ex;
    r = run_schedule(g, p, prof, pol, ex);
  }
  Value out = Value::make_object();
  Value d = Value::make_array();
  for (const auto& rec : r.dispatches) {
    Value x = Value::make_array();
    x.push_back(V(rec.component));
    x.push_back(V(rec.device));
    d.push_back(std::move(x));
  }
  out.set("dispatches", std::move(d));
  Value c = Value::make_array();
  for (const auto& comp : r.completions) {
    Value x = Value::make_array();
    x.push_back(V(comp.component));
    x.push_back(V(comp.event));
    c.push_back(std::move(x));
  }
  out.set("completions", std::move(c));
  out.set("kernel_finish_order", ints(r.kernel_finish_order));
  Scheduler s(g, p, prof, pol);
  Value ranks = Value::make_array();
  for (size_t i = 0; i < s.components().size(); ++i) ranks.push_back(S(s.rank(int(i)).str()));
  out.set("component_ranks", std::move(ranks));
  return out;
}

Ratio ratio_of(const Value& v) { return v.is_string() ? Ratio::parse(v.as_string()) : Ratio(v.as_int64()); }

// {"op":"simulate", spec, params, policy, cpu_devices, callback_delay, heft_waits (0/1), dispatch_cost,
//  "device_profiles": [{"device", "type", "kernel_times": {id: ms}, "kernel_share": {id: s},
//                       "copy_channels", "bandwidth" (bytes/ms), "transfer_latency" (ms)}]}
Value simulate_req(const DagSpec& g, const Value& req) {
  std::set<int> cpu_ids;
  if (const Value* c = req.find("cpu_devices"))
    for (const Value* v : c->items()) cpu_ids.insert(v->as_int());
  Platform p = Platform::from_spec(g, cpu_ids);
  Policy pol = policy_from_name(req.find("policy") ? req.at("policy").as_string() : "clustering");
  std::vector<DeviceProfile> profs;
  for (const Value* d : req.at("device_profiles").items()) {
    DeviceProfile dp;
    dp.device_id = d->at("device").as_int();
    dp.device_type = d->at("type").as_string() == "cpu" ? DeviceType::cpu : DeviceType::gpu;
    if (const Value* t = d->find("kernel_times"))
      for (const auto& [k, v] : t->object_items()) dp.kernel_times[std::stoi(k)] = ratio_of(v);
    if (const Value* t = d->find("kernel_share"))
      for (const auto& [k, v] : t->object_items()) dp.kernel_share[std::stoi(k)] = ratio_of(v);
    if (const Value* v = d->find("copy_channels")) dp.copy_channels = v->as_int();
    if (const Value* v = d->find("bandwidth")) dp.bandwidth = ratio_of(*v);
    if (const Value* v = d->find("transfer_latency")) dp.transfer_latency = ratio_of(*v);
    profs.push_back(std::move(dp));
  }
  const Value* cd = req.find("callback_delay");
  const Value* hw = req.find("heft_waits");
  const Value* dc = req.find("dispatch_cost");
  SimResult r = simulate(g, p, profs, pol, cd ? ratio_of(*cd) : Ratio(0), hw && hw->as_int64() != 0,
                         dc ? ratio_of(*dc) : Ratio(0));
  Value out = Value::make_object();
  out.set("makespan", S(r.makespan.str()));
  out.set("makespan_ms", Value::real(r.makespan.to_double()));
  Value tr = Value::make_array();
  for (const auto& e : r.trace) {
    Value x = Value::make_object();
    x.set("event", V(e.event_id));
    x.set("kind", S(cmd_kind_name(e.kind)));
    x.set("label", S(e.label));
    x.set("kernel", V(e.kernel));
    x.set("component", V(e.component));
    x.set("cmd_event", V(e.cmd_event));
    x.set("device", V(e.device));
    x.set("queue", V(e.queue));
    x.set("channel", V(e.channel));
    x.set("start", S(e.start.str()));
    x.set("finish", S(e.finish.str()));
    tr.push_back(std::move(x));
  }
  out.set("trace", std::move(tr));
  Value d = Value::make_array();
  for (const auto& rec : r.schedule.dispatches) {
    Value x = Value::make_array();
    x.push_back(V(rec.component));
    x.push_back(V(rec.device));
    d.push_back(std::move(x));
  }
  out.set("dispatches", std::move(d));
  out.set("kernel_finish_order", ints(r.schedule.kernel_finish_order));
  return out;
}

Value run(const Value& req) {
  const std::string op = req.at("op").as_string();
  Value out = Value::make_object();
  out.set("ok", Value::boolean(true));
  if (op == "expr") {
    const std::string e = req.at("expr").as_string();
    const Value* m = req.find("mode");
    const std::string mode = m ? m->as_string() : "eval";
    if (mode == "validate") validate_expr(e);
    else if (mode == "positive") out.set("value", V(eval_positive(e, params_of(req))));
    else out.set("value", V(eval_expr(e, params_of(req))));
    return out;
  }
  if (op == "ratio") {
    Ratio a = Ratio::parse(req.at("a").as_string());
    out.set("a", S(a.str()));
    if (req.contains("b")) {
      Ratio b = Ratio::parse(req.at("b").as_string());
      out.set("sum", S((a + b).str()));
      out.set("diff", S((a - b).str()));
      out.set("prod", S((a * b).str()));
      out.set("cmp", V(a < b ? -1 : (a == b ? 0 : 1)));
      out.set("quot", S((a / b).str()));
    }
    return out;
  }
  DagSpec g = parse_spec(req.at("spec").as_string(), params_of(req));
  if (op == "parse") {
    const Value* style = req.find("json_style");
    if (style && style->as_string() == "cudnn-fe")
      out.set("serialized", S(json::dump(spec_to_json(g), 2, json::Style::fe_compact_int_arrays) + "\n"));
    else
      out.set("serialized", S(serialize(g)));
  } else if (op == "analyze") {
    out.set("analysis", analyze(g));
  } else if (op == "ready") {
    std::set<int> fin;
    for (const Value* v : req.at("finished").items()) fin.insert(v->as_int());
    out.set("ready", ints(ready_components(g, derive_components(g), fin)));
  } else if (op == "ranks") {
    std::map<int, Ratio> times;
    for (const auto& [k, v] : req.at("times").object_items()) times[std::stoi(k)] = Ratio::parse(v.as_string());
    auto ranks = bottom_level_ranks(g, [&](int k) { return times.at(k); });
    Value r = Value::make_object();
    for (const auto& [k, v] : ranks) r.set(std::to_string(k), S(v.str()));
    out.set("ranks", std::move(r));
    Value cr = Value::make_array();
    for (const auto& t2 : derive_components(g)) cr.push_back(S(component_rank(t2, ranks).str()));
    out.set("component_ranks", std::move(cr));
  } else if (op == "bytes") {
    Value b = Value::make_array();
    for (const auto& k : g.kernels)
      for (const auto* list : {&k.input_buffers, &k.output_buffers, &k.io_buffers})
        for (const auto& buf : *list) {
          Value x = Value::make_array();
          x.push_back(V(k.id));
          x.push_back(V(buf.pos));
          x.push_back(V(buffer_bytes(buf, g.params)));
          b.push_back(std::move(x));
        }
    out.set("bytes", std::move(b));
  } else if (op == "setup_cq") {
    auto comps = derive_components(g);
    auto ec = classify_edges(g);
    int c = req.at("component").as_int();
    if (c < 0 || size_t(c) >= comps.size()) fail(Errc::invalid_param, "component out of range");
    const Value* dt = req.find("device_type");
    DeviceType type = (dt && dt->as_string() == "cpu") ? DeviceType::cpu : DeviceType::gpu;
    int dev = req.find("device") ? req.at("device").as_int() : 0;
    int r = req.at("queues").as_int();
    auto q = setup_cq(comps[size_t(c)], dev, type, r, g, ec);
    out.set("cq", json::parse(to_debug_json(q)));
  } else if (op == "schedule") {
    out.set("schedule", schedule(g, req));
  } else if (op == "simulate") {
    out.set("simulate", simulate_req(g, req));
  } else {
    fail(Errc::invalid_param, "unknown op " + op);
  }
  return out;
}

char* dup_string(const std::string& s) {
  char* buf = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return buf;
}

}  // namespace

extern "C" char* hs_query(const char* request) {
  Value out;
  auto error = [&](const char* name, int exit_code, const std::string& msg) {
    out = Value::make_object();
    out.set("ok", Value::boolean(false));
    out.set("errc", S(name));
    if (exit_code >= 0) out.set("exit", V(exit_code));
    out.set("message", S(msg));
  };
  try {
    out = run(json::parse(request ? request : ""));
  } catch (const Error& e) {
    error(errc_name(e.code()), exit_code_for(e.code()), e.what());
  } catch (const std::exception& e) {
    error("StdException", -1, e.what());
  }
  return dup_string(json::dump(out, -1));
}

extern "C" void hs_free_string(char* s) { std::free(s); }
