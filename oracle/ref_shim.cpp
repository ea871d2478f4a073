// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI shim over the *reference's own* hetsim L0-L2 sources, compiled
// straight from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libhetsim_ref.so. It answers the same JSON queries as the
// product's `hs_query` (paper_2009_07482_b200/csrc/capi/query.cpp) so the
// differential tests in tests/ can compare the two implementations on
// identical inputs. Queries implemented here only touch functions that the
// reference actually implements (errors, rational, expr, spec_model,
// graph_analysis); cq_builder/scheduler have no reference implementation.
#include <cstdlib>
#include <cstring>
#include <string>

#include <json.hpp>

#include "hetsim/errors.hpp"
#include "hetsim/expr.hpp"
#include "hetsim/graph_analysis.hpp"
#include "hetsim/rational.hpp"
#include "hetsim/spec_model.hpp"

using nlohmann::ordered_json;
using namespace hetsim;

namespace {

ParamMap params_of(const ordered_json& req) {
  ParamMap p;
  if (req.contains("params"))
    for (auto it = req["params"].begin(); it != req["params"].end(); ++it) p[it.key()] = it.value().get<long long>();
  return p;
}

ordered_json set_json(const std::set<int>& s) {
  ordered_json a = ordered_json::array();
  for (int v : s) a.push_back(v);
  return a;
}

ordered_json analyze(const DagSpec& g) {
  ordered_json out;
  out["topo_order"] = g.topo_order();
  ordered_json comps = ordered_json::array();
  for (const auto& t : derive_components(g)) {
    ordered_json c;
    c["id"] = t.id;
    c["kernels"] = t.kernel_ids;
    c["dev_pref"] = device_type_name(t.dev_pref);
    c["front"] = set_json(t.front);
    c["end"] = set_json(t.end);
    c["interior"] = set_json(t.interior);
    comps.push_back(c);
  }
  out["components"] = comps;
  auto ec = classify_edges(g);
  ordered_json kinds = ordered_json::array();
  for (auto k : ec.edge_kind) kinds.push_back(k == EdgeKind::intra ? "intra" : "inter");
  out["edge_kind"] = kinds;
  ordered_json wc = ordered_json::array(), rc = ordered_json::array();
  for (const auto& [key, cls] : ec.write_class)
    wc.push_back({key.first, key.second, cls == CopyClass::isolated ? "isolated" : "dependent"});
  for (const auto& [key, cls] : ec.read_class)
    rc.push_back({key.first, key.second, cls == CopyClass::isolated ? "isolated" : "dependent"});
  out["write_class"] = wc;
  out["read_class"] = rc;
  ordered_json succ = ordered_json::array();
  for (const auto& [k, s] : g.kernel_successors()) succ.push_back({k, set_json(s)});
  out["successors"] = succ;
  ordered_json comp_of = ordered_json::array();
  for (const auto& [k, c] : g.component_of()) comp_of.push_back({k, c});
  out["component_of"] = comp_of;
  return out;
}

ordered_json run(const ordered_json& req) {
  const std::string op = req.at("op").get<std::string>();
  ordered_json out;
  out["ok"] = true;
  if (op == "expr") {
    const std::string e = req.at("expr").get<std::string>();
    const std::string mode = req.value("mode", "eval");
    if (mode == "validate") {
      validate_expr(e);
    } else if (mode == "positive") {
      out["value"] = eval_positive(e, params_of(req));
    } else {
      out["value"] = eval_expr(e, params_of(req));
    }
    return out;
  }
  if (op == "ratio") {
    Ratio a = Ratio::parse(req.at("a").get<std::string>());
    out["a"] = a.str();
    if (req.contains("b")) {
      Ratio b = Ratio::parse(req.at("b").get<std::string>());
      out["sum"] = (a + b).str();
      out["diff"] = (a - b).str();
      out["prod"] = (a * b).str();
      out["cmp"] = a < b ? -1 : (a == b ? 0 : 1);
      out["quot"] = (a / b).str();
    }
    return out;
  }
  DagSpec g = parse_spec(req.at("spec").get<std::string>(), params_of(req));
  if (op == "parse") {
    out["serialized"] = serialize(g);
  } else if (op == "analyze") {
    out["analysis"] = analyze(g);
  } else if (op == "ready") {
    std::set<int> fin;
    for (const auto& v : req.at("finished")) fin.insert(v.get<int>());
    out["ready"] = ready_components(g, derive_components(g), fin);
  } else if (op == "ranks") {
    std::map<int, Ratio> times;
    for (auto it = req.at("times").begin(); it != req.at("times").end(); ++it)
      times[std::stoi(it.key())] = Ratio::parse(it.value().get<std::string>());
    auto ranks = bottom_level_ranks(g, [&](int k) { return times.at(k); });
    ordered_json r = ordered_json::object();
    for (const auto& [k, v] : ranks) r[std::to_string(k)] = v.str();
    out["ranks"] = r;
    ordered_json cr = ordered_json::array();
    for (const auto& t : derive_components(g)) cr.push_back(component_rank(t, ranks).str());
    out["component_ranks"] = cr;
  } else if (op == "bytes") {
    ordered_json b = ordered_json::array();
    for (const auto& k : g.kernels)
      for (const auto* list : {&k.input_buffers, &k.output_buffers, &k.io_buffers})
        for (const auto& buf : *list) b.push_back({k.id, buf.pos, buffer_bytes(buf, g.params)});
    out["bytes"] = b;
  } else {
    out["ok"] = false;
    out["errc"] = "InvalidParam";
    out["message"] = "unknown op " + op;
  }
  return out;
}

}  // namespace

extern "C" {

// Returns a malloc'd JSON string; free with ref_free.
char* ref_query(const char* request) {
  ordered_json out;
  try {
    out = run(ordered_json::parse(request));
  } catch (const Error& e) {
    out = ordered_json::object();
    out["ok"] = false;
    out["errc"] = errc_name(e.code());
    out["exit"] = exit_code_for(e.code());
    out["message"] = e.what();
  } catch (const std::exception& e) {
    out = ordered_json::object();
    out["ok"] = false;
    out["errc"] = "StdException";
    out["message"] = e.what();
  }
  std::string s = out.dump();
  char* buf = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return buf;
}

void ref_free(char* p) { std::free(p); }

}  // extern "C"
