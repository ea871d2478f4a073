// hetsim-b200 — Alg. 1 scheduler (schedule / select / dispatch / cb).
//
// The reference specifies this module only in prose (SPEC.md:278-368,
// PAPER.md:253-289, 312-316). The dispatch entry point is the `Executor`
// interface: the scheduler hands it (T, Q) pairs exactly where Alg. 1 calls
// dispatch(), and the executor reports callback-marked command completions
// back (Alg. 1 cb). Implementations in this repo:
//   * PlanExecutor    — deterministic completion model (dispatch order); used to
//                       derive the static plan that is captured as a CUDA graph.
//   * ReplayExecutor  — replays a recorded completion log (scheduling parity).
//   * CudaExecutor    — real streams/events/kernels on the B200
//                       (include/hetsim/cuda_executor.hpp).
#pragma once

#include <deque>
#include <map>
#include <memory>
#include <optional>
#include <set>
#include <string>
#include <utility>
#include <vector>

#include "hetsim/cq_builder.hpp"
#include "hetsim/graph_analysis.hpp"
#include "hetsim/rational.hpp"
#include "hetsim/spec_model.hpp"

namespace hetsim {

enum class Policy { clustering, eager, heft };
const char* policy_name(Policy p);
Policy policy_from_name(const std::string& name);  // InvalidParam

struct DeviceInfo {
  int id = -1;
  DeviceType type = DeviceType::gpu;
  int queues = 1;
  int gpu_ordinal = 0;  // physical GPU for type gpu (logical devices may share one)
};

struct Platform {
  std::vector<DeviceInfo> devices;  // ascending id
  /// Devices from the spec's cq map; ids listed in `cpu_ids` are CPU devices,
  /// all others GPU devices mapped round-robin onto `n_gpus` physical GPUs.
  static Platform from_spec(const DagSpec& g, const std::set<int>& cpu_ids = {}, int n_gpus = 1);
  const DeviceInfo& device(int id) const;  // InvalidParam
};

/// Standalone kernel times per device type. Empty = unit times.
struct Profiles {
  std::map<std::pair<int, DeviceType>, Ratio> time;
  Ratio time_of(int kernel, DeviceType t) const;  // MissingProfileEntry
  bool empty() const { return time.empty(); }
};

/// A callback-marked event of a dispatched component has completed.
struct Completion {
  int component = -1;
  int event = -1;
};

class Executor {
 public:
  virtual ~Executor() = default;
  /// Alg. 1 dispatch(): submit every queue of `q` (the device is locked to
  /// `t` until the scheduler sees all of its terminal events complete).
  virtual void dispatch(const TaskComponent& t, const CommandQueueStructure& q) = 0;
  /// Blocks until the next callback-marked event completes (Alg. 1
  /// sleep_till_cb_update + cb delivery). Raises Deadlock if none can.
  virtual Completion wait_next() = 0;
  /// The executor's clock (ms), when it has one (the platform simulator); HEFT's
  /// busy-device mode estimates release times from it.
  virtual std::optional<Ratio> clock() const { return std::nullopt; }
};

struct DispatchRecord {
  int component = -1;
  int device = -1;
};

struct ScheduleResult {
  std::vector<DispatchRecord> dispatches;        // in dispatch order
  std::vector<Completion> completions;           // in delivery order
  std::vector<int> kernel_finish_order;          // kernels as the scheduler saw them finish
  std::vector<CommandQueueStructure> structures; // per dispatch, same order as dispatches
};

class Scheduler {
 public:
  Scheduler(const DagSpec& g, Platform platform, Profiles profiles, Policy policy);

  ScheduleResult run(Executor& ex);

  /// HEFT busy-device mode (`--heft-waits`): select() also weighs
  /// busy devices, EFT(k, d) = remaining time of d's component + t(k, d), and
  /// waits for a busy device that wins. Default off (strict availability).
  void set_heft_waits(bool on) { heft_waits_ = on; }

  const std::vector<TaskComponent>& components() const { return comps_; }
  const EdgeClasses& edge_classes() const { return ec_; }
  const Ratio& rank(int component) const { return comp_rank_.at(size_t(component)); }

  /// One select() call over the current F/A (exposed for unit tests).
  std::optional<std::pair<int, int>> select(const std::set<int>& frontier, const std::set<int>& available) const;

 private:
  enum class State { waiting, queued, dispatched, done };
  void cb(const Completion& c, ScheduleResult& out);
  void mark_finished(int kernel, ScheduleResult& out);
  void enqueue_ready(std::set<int>& frontier);
  Ratio component_time(int comp, DeviceType t) const;

  const DagSpec& g_;
  Platform platform_;
  Profiles profiles_;
  Policy policy_;
  std::vector<TaskComponent> comps_;
  EdgeClasses ec_;
  std::vector<Ratio> comp_rank_;
  std::vector<std::vector<int>> cross_preds_;  // per component: kernels of other components it waits for
  std::map<int, int> comp_of_;

  // HEFT with busy devices: the max-rank component's device by EFT over every
  // device at time `now` (none if that device is busy: wait for it)
  std::optional<std::pair<int, int>> select_heft_waits(const Ratio& now) const;
  bool heft_waits_ = false;

  // run state
  std::vector<State> state_;
  std::set<int> finished_;
  std::set<int> frontier_, available_;
  struct Live {
    int device = -1;
    CommandQueueStructure q;
    std::set<int> done_events;
    Ratio release;  // dispatch time + profiled component time (heft_waits)
  };
  std::map<int, Live> live_;
};

ScheduleResult run_schedule(const DagSpec& g, const Platform& p, const Profiles& prof, Policy policy, Executor& ex,
                            bool heft_waits = false);

/// Completion model used to build static (graph-captured) plans: components
/// complete in dispatch order, each reporting its callback events in event order.
class PlanExecutor : public Executor {
 public:
  void dispatch(const TaskComponent& t, const CommandQueueStructure& q) override;
  Completion wait_next() override;

 private:
  std::deque<Completion> pending_;
};

/// Re-delivers a recorded completion log (e.g. captured from a GPU run).
class ReplayExecutor : public Executor {
 public:
  explicit ReplayExecutor(std::vector<Completion> log) : log_(std::move(log)) {}
  void dispatch(const TaskComponent& t, const CommandQueueStructure& q) override;
  Completion wait_next() override;

 private:
  std::vector<Completion> log_;
  size_t next_ = 0;
  std::set<int> dispatched_;
};

}  // namespace hetsim
