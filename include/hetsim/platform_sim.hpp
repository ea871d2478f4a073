// hetsim-b200 — platform_sim: the deterministic discrete-event platform model of
// SPEC.md:370-440 (the reference specifies it in prose only).
//
// On the B200 the real executor (streams, copy engines, hardware kernel
// concurrency) replaces it for execution; this model is kept for what the
// SURVEY (§8f row 3) asks of it: a CPU-side cost model that can be fed with
// kernel times measured on the GPU and compared with measured makespans, and
// the policy/partition studies of the paper without a GPU.
//
// Semantics:
//  * a command is runnable when every earlier command of its queue finished,
//    every E_Q predecessor finished and a resource is available;
//  * transfers take transfer_latency + bytes / bandwidth on a GPU (0 on a CPU)
//    on the least-loaded copy channel (earliest free time, ties -> lower id),
//    FIFO per channel;
//  * ndranges of one device share it: with running set S and sigma = sum of
//    their shares, each progresses at rate 1 (sigma <= 1) or 1/sigma;
//  * simultaneous completions complete in (device, queue, position) order;
//    callback-marked completions reach the scheduler `callback_delay` later;
//  * host dispatch cost (B200 extension, profiles/sim_vs_measured.py): issuing a
//    component occupies the host thread for `dispatch_cost`, one component at a
//    time; its commands cannot start before the host has issued it.
// Time is an exact rational (milliseconds): identical inputs give
// bit-identical traces.
#pragma once

#include <map>
#include <string>
#include <vector>

#include "hetsim/cq_builder.hpp"
#include "hetsim/rational.hpp"
#include "hetsim/scheduler.hpp"

namespace hetsim {

struct DeviceProfile {
  int device_id = -1;
  DeviceType device_type = DeviceType::gpu;
  std::map<int, Ratio> kernel_times;  // kernel id -> standalone ms (> 0)
  std::map<int, Ratio> kernel_share;  // kernel id -> compute share in (0,1]; default 1
  int copy_channels = 2;
  Ratio bandwidth = Ratio(1);         // bytes per ms (> 0)
  Ratio transfer_latency = Ratio(0);  // ms (>= 0)
};

/// transfer_time(bytes, d).
Ratio transfer_time(int64_t bytes, const DeviceProfile& d);

struct SimEvent {
  int event_id = -1;  // completion order
  int component = -1;
  int cmd_event = -1;  // the command's event id inside its component's CQS
  CmdKind kind = CmdKind::ndrange;
  std::string label;
  int kernel = -1;
  int device = -1;
  int queue = -1;
  int channel = -1;  // copy channel of a GPU transfer, -1 otherwise
  Ratio start, finish;
};

class PlatformSim : public Executor {
 public:
  /// profiles: one per logical device of the spec's cq map (InvalidParam if missing).
  PlatformSim(std::vector<DeviceProfile> profiles, Ratio callback_delay = Ratio(0), Ratio dispatch_cost = Ratio(0));

  void dispatch(const TaskComponent& t, const CommandQueueStructure& q) override;
  Completion wait_next() override;  // SimDeadlock when commands remain but none can run

  const std::vector<SimEvent>& trace() const { return trace_; }
  Ratio now() const { return now_; }
  std::optional<Ratio> clock() const override { return now_; }
  Ratio makespan() const;  // EmptyTrace

  /// Scheduler profiles (per device type) implied by the device profiles.
  static Profiles scheduler_profiles(const std::vector<DeviceProfile>& profiles);

 private:
  enum class St { pending, running, done };
  struct Cmd {
    int comp = -1, ev = -1, device = -1, queue = -1, pos = -1, kernel = -1, channel = -1;
    CmdKind kind = CmdKind::ndrange;
    std::string label;
    int64_t bytes = 0;
    bool callback = false;
    std::vector<int> preds;  // indices into cmds_
    int queue_prev = -1;     // index of the previous command in the same queue
    St st = St::pending;
    Ratio start, finish, remaining;
    Ratio ready_at;  // earliest start: the host has issued the component
  };
  const DeviceProfile& prof(int device) const;
  void start_runnable();
  Ratio rate(int device) const;
  bool next_completion(Ratio* t, int* idx) const;

  std::map<int, DeviceProfile> profiles_;
  Ratio callback_delay_;
  Ratio dispatch_cost_;
  Ratio host_free_ = Ratio(0);  // the host thread issues one component at a time
  Ratio now_ = Ratio(0);
  std::vector<Cmd> cmds_;
  std::map<int, std::vector<Ratio>> channel_free_;  // device -> per-channel free time
  std::vector<std::pair<Ratio, Completion>> deliveries_;  // FIFO within equal times
  std::vector<SimEvent> trace_;
};

/// Alg. 1 over the simulated platform: the scheduler uses the profiles' kernel
/// times for ranks / HEFT and the simulator as its executor.
struct SimResult {
  ScheduleResult schedule;
  std::vector<SimEvent> trace;
  Ratio makespan;
};
SimResult simulate(const DagSpec& g, const Platform& p, const std::vector<DeviceProfile>& profiles, Policy policy,
                   Ratio callback_delay = Ratio(0), bool heft_waits = false, Ratio dispatch_cost = Ratio(0));

}  // namespace hetsim
