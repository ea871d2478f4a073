// platform_sim: see include/hetsim/platform_sim.hpp.
#include "hetsim/platform_sim.hpp"

#include <algorithm>
#include <tuple>

#include "hetsim/errors.hpp"

namespace hetsim {

Ratio transfer_time(int64_t bytes, const DeviceProfile& d) {
  if (d.device_type == DeviceType::cpu) return Ratio(0);
  return d.transfer_latency + Ratio(static_cast<long long>(bytes)) / d.bandwidth;
}

PlatformSim::PlatformSim(std::vector<DeviceProfile> profiles, Ratio callback_delay, Ratio dispatch_cost)
    : callback_delay_(callback_delay), dispatch_cost_(dispatch_cost) {
  if (callback_delay < Ratio(0)) fail(Errc::invalid_param, "callback delay must be >= 0");
  if (dispatch_cost < Ratio(0)) fail(Errc::invalid_param, "dispatch cost must be >= 0");
  for (auto& p : profiles) {
    if (profiles_.count(p.device_id)) fail(Errc::invalid_param, "duplicate profile for device " + std::to_string(p.device_id));
    if (p.device_type == DeviceType::gpu && p.copy_channels < 1)
      fail(Errc::invalid_param, "device " + std::to_string(p.device_id) + ": copy_channels must be >= 1");
    if (p.device_type == DeviceType::gpu && !(Ratio(0) < p.bandwidth))
      fail(Errc::invalid_param, "device " + std::to_string(p.device_id) + ": bandwidth must be > 0");
    for (const auto& [k, t] : p.kernel_times)
      if (!(Ratio(0) < t)) fail(Errc::invalid_param, "kernel " + std::to_string(k) + ": time must be > 0");
    for (const auto& [k, s] : p.kernel_share)
      if (!(Ratio(0) < s) || Ratio(1) < s) fail(Errc::invalid_param, "kernel " + std::to_string(k) + ": share not in (0,1]");
    channel_free_[p.device_id] = std::vector<Ratio>(size_t(std::max(1, p.copy_channels)), Ratio(0));
    const int id = p.device_id;
    profiles_.emplace(id, std::move(p));
  }
}

const DeviceProfile& PlatformSim::prof(int device) const {
  auto it = profiles_.find(device);
  if (it == profiles_.end()) fail(Errc::missing_profile_entry, "no profile for device " + std::to_string(device));
  return it->second;
}

Profiles PlatformSim::scheduler_profiles(const std::vector<DeviceProfile>& profiles) {
  Profiles out;
  for (const auto& p : profiles)
    for (const auto& [k, t] : p.kernel_times) out.time.emplace(std::make_pair(k, p.device_type), t);
  return out;
}

void PlatformSim::dispatch(const TaskComponent& t, const CommandQueueStructure& q) {
  prof(q.device);
  host_free_ = rmax(now_, host_free_) + dispatch_cost_;
  std::map<int, int> idx_of;  // event -> index into cmds_
  for (size_t qi = 0; qi < q.queues.size(); ++qi) {
    int prev = -1;
    for (size_t i = 0; i < q.queues[qi].size(); ++i) {
      const Command& c = q.queues[qi][i];
      Cmd m;
      m.comp = t.id;
      m.ev = c.event;
      m.device = q.device;
      m.queue = int(qi);
      m.pos = int(i);
      m.kernel = c.kernel;
      m.kind = c.kind;
      m.label = c.label;
      m.bytes = c.bytes;
      m.callback = q.callbacks.count(c.event) > 0;
      m.queue_prev = prev;
      m.ready_at = host_free_;
      prev = int(cmds_.size());
      idx_of[c.event] = prev;
      cmds_.push_back(std::move(m));
    }
  }
  for (auto [a, b] : q.deps) cmds_[size_t(idx_of.at(b))].preds.push_back(idx_of.at(a));
}

Ratio PlatformSim::rate(int device) const {
  Ratio sigma(0);
  for (const auto& c : cmds_)
    if (c.st == St::running && c.kind == CmdKind::ndrange && c.device == device) {
      const auto& sh = prof(device).kernel_share;
      auto it = sh.find(c.kernel);
      sigma += it == sh.end() ? Ratio(1) : it->second;
    }
  return sigma <= Ratio(1) ? Ratio(1) : Ratio(1) / sigma;
}

void PlatformSim::start_runnable() {
  // deterministic order: (device, queue, position, component)
  std::vector<int> order;
  for (size_t i = 0; i < cmds_.size(); ++i)
    if (cmds_[i].st == St::pending) order.push_back(int(i));
  std::sort(order.begin(), order.end(), [&](int a, int b) {
    const Cmd &x = cmds_[size_t(a)], &y = cmds_[size_t(b)];
    return std::tie(x.device, x.queue, x.pos, x.comp) < std::tie(y.device, y.queue, y.pos, y.comp);
  });
  for (int i : order) {
    Cmd& c = cmds_[size_t(i)];
    if (now_ < c.ready_at) continue;
    if (c.queue_prev >= 0 && cmds_[size_t(c.queue_prev)].st != St::done) continue;
    bool ready = true;
    for (int p : c.preds) ready = ready && cmds_[size_t(p)].st == St::done;
    if (!ready) continue;
    const DeviceProfile& d = prof(c.device);
    c.st = St::running;
    if (c.kind == CmdKind::ndrange) {
      auto it = d.kernel_times.find(c.kernel);
      if (it == d.kernel_times.end())
        fail(Errc::missing_profile_entry, "kernel " + std::to_string(c.kernel) + " has no time on device " +
                                              std::to_string(c.device));
      c.start = now_;
      c.remaining = it->second;
    } else if (d.device_type == DeviceType::cpu) {
      c.start = c.finish = now_;
    } else {
      auto& free = channel_free_.at(c.device);
      size_t ch = 0;
      for (size_t k = 1; k < free.size(); ++k)
        if (free[k] < free[ch]) ch = k;
      c.channel = int(ch);
      c.start = rmax(now_, free[ch]);
      c.finish = c.start + transfer_time(c.bytes, d);
      free[ch] = c.finish;
    }
  }
}

bool PlatformSim::next_completion(Ratio* t, int* idx) const {
  bool found = false;
  std::map<int, Ratio> rates;
  for (size_t i = 0; i < cmds_.size(); ++i) {
    const Cmd& c = cmds_[i];
    if (c.st != St::running) continue;
    Ratio f;
    if (c.kind == CmdKind::ndrange) {
      auto r = rates.find(c.device);
      if (r == rates.end()) r = rates.emplace(c.device, rate(c.device)).first;
      f = now_ + c.remaining / r->second;
    } else {
      f = c.finish;
    }
    if (!found || f < *t ||
        (f == *t && std::tie(c.device, c.queue, c.pos, c.comp) <
                        std::tie(cmds_[size_t(*idx)].device, cmds_[size_t(*idx)].queue, cmds_[size_t(*idx)].pos,
                                 cmds_[size_t(*idx)].comp))) {
      *t = f;
      *idx = int(i);
      found = true;
    }
  }
  return found;
}

Completion PlatformSim::wait_next() {
  auto advance_to = [&](const Ratio& t) {
    if (t == now_) return;
    std::map<int, Ratio> rates;
    for (auto& c : cmds_)
      if (c.st == St::running && c.kind == CmdKind::ndrange) {
        auto r = rates.find(c.device);
        if (r == rates.end()) r = rates.emplace(c.device, rate(c.device)).first;
        c.remaining -= r->second * (t - now_);
      }
    now_ = t;
  };
  for (;;) {
    start_runnable();
    Ratio tc;
    int idx = -1;
    const bool has = next_completion(&tc, &idx);
    size_t di = deliveries_.size();
    for (size_t i = 0; i < deliveries_.size(); ++i)
      if (di == deliveries_.size() || deliveries_[i].first < deliveries_[di].first) di = i;
    // the next moment the host finishes issuing a component whose commands wait for it
    bool has_rel = false;
    Ratio rel;
    for (const auto& c : cmds_)
      if (c.st == St::pending && now_ < c.ready_at && (!has_rel || c.ready_at < rel)) {
        rel = c.ready_at;
        has_rel = true;
      }
    if (has_rel && (!has || rel < tc) && (di == deliveries_.size() || rel <= deliveries_[di].first)) {
      advance_to(rel);
      continue;
    }
    // completions at time T are processed before callbacks delivered at T
    if (di < deliveries_.size() && (!has || deliveries_[di].first < tc)) {
      advance_to(rmax(now_, deliveries_[di].first));
      Completion c = deliveries_[di].second;
      deliveries_.erase(deliveries_.begin() + long(di));
      return c;
    }
    if (!has) {
      for (const auto& c : cmds_)
        if (c.st == St::pending)
          fail(Errc::sim_deadlock, "command " + c.label + " of component " + std::to_string(c.comp) + " can never run");
      fail(Errc::deadlock, "no outstanding events");
    }
    advance_to(tc);
    Cmd& c = cmds_[size_t(idx)];
    c.st = St::done;
    c.finish = now_;
    c.remaining = Ratio(0);
    SimEvent e;
    e.event_id = int(trace_.size());
    e.component = c.comp;
    e.cmd_event = c.ev;
    e.kind = c.kind;
    e.label = c.label;
    e.kernel = c.kernel;
    e.device = c.device;
    e.queue = c.queue;
    e.channel = c.channel;
    e.start = c.start;
    e.finish = c.finish;
    trace_.push_back(e);
    if (c.callback) deliveries_.push_back({now_ + callback_delay_, Completion{c.comp, c.ev}});
  }
}

Ratio PlatformSim::makespan() const {
  if (trace_.empty()) fail(Errc::empty_trace, "trace has no events");
  Ratio a = trace_.front().start, b = trace_.front().finish;
  for (const auto& e : trace_) {
    a = rmin(a, e.start);
    b = rmax(b, e.finish);
  }
  return b - a;
}

SimResult simulate(const DagSpec& g, const Platform& p, const std::vector<DeviceProfile>& profiles, Policy policy,
                   Ratio callback_delay, bool heft_waits, Ratio dispatch_cost) {
  for (const auto& d : p.devices) {
    auto it = std::find_if(profiles.begin(), profiles.end(), [&](const DeviceProfile& x) { return x.device_id == d.id; });
    if (it == profiles.end()) fail(Errc::missing_profile_entry, "no profile for device " + std::to_string(d.id));
    if (it->device_type != d.type)
      fail(Errc::invalid_param, "device " + std::to_string(d.id) + ": profile type does not match the platform");
  }
  Scheduler sched(g, p, PlatformSim::scheduler_profiles(profiles), policy);
  sched.set_heft_waits(heft_waits);
  PlatformSim sim(profiles, callback_delay, dispatch_cost);
  SimResult r;
  r.schedule = sched.run(sim);
  r.trace = sim.trace();
  r.makespan = sim.makespan();
  return r;
}

}  // namespace hetsim
