// Source-level drop-in check: a C++ caller written against the reference's
// headers (proj/include/hetsim/spec_model.hpp:90-95 parse_spec,
// graph_analysis.hpp:27-38 derive_components) plus the scheduler / executor
// plug-in, linked against libhetsim.so, runs a DAG on the B200.
//
//   dropin_main SPEC PARAMS IO_IN IO_OUT N BATCH [POLICY]
// PARAMS: "NAME VALUE" lines. IO_IN: records {int32 kernel, int32 pos, int32
// is_output, int64 stride_bytes, int64 count, int64 nbytes, bytes}; outputs
// (is_output = 1, zero-filled) are written to IO_OUT in the same format.
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "hetsim/cuda_executor.hpp"
#include "hetsim/errors.hpp"
#include "hetsim/graph_analysis.hpp"
#include "hetsim/scheduler.hpp"
#include "hetsim/spec_model.hpp"

struct Rec {
  int32_t kernel, pos, is_output;
  int64_t stride, count;
  std::vector<char> data;
};

int main(int argc, char** argv) {
  if (argc != 7 && argc != 8) {
    std::cerr << "usage: dropin_main SPEC PARAMS IO_IN IO_OUT N BATCH [POLICY]\n";
    return 2;
  }
  try {
    std::ifstream sf(argv[1]);
    std::stringstream ss;
    ss << sf.rdbuf();
    hetsim::ParamMap params;
    std::ifstream pf(argv[2]);
    std::string name;
    long long v;
    while (pf >> name >> v) params[name] = v;
    const hetsim::DagSpec g = hetsim::parse_spec(ss.str(), params);
    const auto comps = hetsim::derive_components(g);

    std::ifstream in(argv[3], std::ios::binary);
    std::vector<Rec> recs;
    for (;;) {
      Rec r;
      int64_t nbytes = 0;
      if (!in.read(reinterpret_cast<char*>(&r.kernel), 4)) break;
      in.read(reinterpret_cast<char*>(&r.pos), 4);
      in.read(reinterpret_cast<char*>(&r.is_output), 4);
      in.read(reinterpret_cast<char*>(&r.stride), 8);
      in.read(reinterpret_cast<char*>(&r.count), 8);
      in.read(reinterpret_cast<char*>(&nbytes), 8);
      r.data.resize(size_t(nbytes));
      in.read(r.data.data(), nbytes);
      recs.push_back(std::move(r));
    }
    const int64_t n = std::stoll(argv[5]);
    hetsim::CudaExecutorOptions opts;
    opts.batch = std::stoi(argv[6]);
    hetsim::CudaExecutor ex(g, opts);
    for (auto& r : recs) ex.bind(r.kernel, r.pos, r.data.data(), r.stride, r.count);
    const hetsim::Platform platform = hetsim::Platform::from_spec(g);
    const hetsim::Policy policy = argc == 8 ? hetsim::policy_from_name(argv[7]) : hetsim::Policy::clustering;
    int64_t total_ns = 0;
    size_t dispatches = 0;
    for (int64_t first = 0; first < n; first += opts.batch) {
      const int64_t cnt = std::min<int64_t>(opts.batch, n - first);
      ex.begin(first, cnt);
      const hetsim::ScheduleResult res =
          hetsim::run_schedule(g, platform, hetsim::Profiles{}, policy, ex);
      total_ns += ex.end();
      dispatches = res.dispatches.size();
    }
    std::ofstream out(argv[4], std::ios::binary);
    for (const auto& r : recs) {
      if (!r.is_output) continue;
      const int64_t nbytes = int64_t(r.data.size());
      out.write(reinterpret_cast<const char*>(&r.kernel), 4);
      out.write(reinterpret_cast<const char*>(&r.pos), 4);
      out.write(reinterpret_cast<const char*>(&r.is_output), 4);
      out.write(reinterpret_cast<const char*>(&r.stride), 8);
      out.write(reinterpret_cast<const char*>(&r.count), 8);
      out.write(reinterpret_cast<const char*>(&nbytes), 8);
      out.write(r.data.data(), nbytes);
    }
    std::printf("components %zu dispatches %zu device_ns %lld\n", comps.size(), dispatches,
                static_cast<long long>(total_ns));
    return 0;
  } catch (const hetsim::Error& e) {
    std::cerr << e.what() << "\n";
    return hetsim::exit_code_for(e.code());
  }
}
