// Alg. 1 — schedule / select / cb.
//
// Single-threaded event loop: the executor may deliver completions from
// other threads (CUDA host callbacks push onto its queue), but cb() itself
// always runs on the scheduler thread, which is the spec's "each handler runs
// to completion" form of the paper's lock()/unlock().
//
// Decisions:
//  * readiness = every cross-component predecessor kernel finished;
//  * GPU END kernel finished when all of its dependent reads completed, CPU
//    END kernel when its ndrange completed;
//  * component finished (device returned) when the terminal command of every
//    queue completed;
//  * clustering: max rank, ties lower component id then lower device id;
//    eager: max rank on the lowest-id available device;
//    heft: max rank on the available device with minimal EFT, ties lower id;
//    heft with heft_waits: EFT over every device, a busy one counting the residual
//    time of its component (release = dispatch time + profiled time), and a busy
//    winner is waited for.
#include "hetsim/scheduler.hpp"

#include <algorithm>

#include "hetsim/errors.hpp"

namespace hetsim {

const char* policy_name(Policy p) {
  switch (p) {
    case Policy::clustering: return "clustering";
    case Policy::eager: return "eager";
    case Policy::heft: return "heft";
  }
  return "?";
}

Policy policy_from_name(const std::string& name) {
  if (name == "clustering") return Policy::clustering;
  if (name == "eager") return Policy::eager;
  if (name == "heft") return Policy::heft;
  fail(Errc::invalid_param, "unknown policy '" + name + "'");
}

Platform Platform::from_spec(const DagSpec& g, const std::set<int>& cpu_ids, int n_gpus) {
  Platform p;
  int gpu_seq = 0;
  for (const auto& [id, n] : g.cq) {
    DeviceInfo d;
    d.id = id;
    d.queues = n;
    d.type = cpu_ids.count(id) ? DeviceType::cpu : DeviceType::gpu;
    d.gpu_ordinal = d.type == DeviceType::gpu ? (gpu_seq++ % std::max(1, n_gpus)) : -1;
    p.devices.push_back(d);
  }
  return p;
}

const DeviceInfo& Platform::device(int id) const {
  for (const auto& d : devices)
    if (d.id == id) return d;
  fail(Errc::invalid_param, "unknown device " + std::to_string(id));
}

Ratio Profiles::time_of(int kernel, DeviceType t) const {
  auto it = time.find({kernel, t});
  if (it == time.end())
    fail(Errc::missing_profile_entry,
         "kernel " + std::to_string(kernel) + " on " + device_type_name(t) + " has no profile time");
  return it->second;
}

Scheduler::Scheduler(const DagSpec& g, Platform platform, Profiles profiles, Policy policy)
    : g_(g), platform_(std::move(platform)), profiles_(std::move(profiles)), policy_(policy) {
  comps_ = derive_components(g_);
  ec_ = classify_edges(g_);
  comp_of_ = g_.component_of();
  auto ranks = bottom_level_ranks(g_, [&](int k) -> Ratio {
    return profiles_.empty() ? Ratio(1) : profiles_.time_of(k, g_.kernel(k).dev);
  });
  comp_rank_.reserve(comps_.size());
  for (const auto& t : comps_) comp_rank_.push_back(component_rank(t, ranks));
  cross_preds_.assign(comps_.size(), {});
  for (const auto& e : g_.edges) {
    int cs = comp_of_.at(e.src_kernel), cd = comp_of_.at(e.dst_kernel);
    if (cs != cd) cross_preds_[size_t(cd)].push_back(e.src_kernel);
  }
  for (auto& v : cross_preds_) {
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
  }
}

Ratio Scheduler::component_time(int comp, DeviceType t) const {
  Ratio sum = 0;
  for (int k : comps_[size_t(comp)].kernel_ids) sum += profiles_.empty() ? Ratio(1) : profiles_.time_of(k, t);
  return sum;
}

std::optional<std::pair<int, int>> Scheduler::select(const std::set<int>& frontier,
                                                     const std::set<int>& available) const {
  if (frontier.empty() || available.empty()) return std::nullopt;
  // Frontier in priority order: rank descending, component id ascending.
  std::vector<int> order(frontier.begin(), frontier.end());
  std::stable_sort(order.begin(), order.end(),
                   [&](int a, int b) { return comp_rank_[size_t(b)] < comp_rank_[size_t(a)]; });
  switch (policy_) {
    case Policy::clustering:
      for (int c : order)
        for (int d : available)
          if (platform_.device(d).type == comps_[size_t(c)].dev_pref) return std::make_pair(c, d);
      return std::nullopt;
    case Policy::eager:
      return std::make_pair(order.front(), *available.begin());
    case Policy::heft: {
      int c = order.front();
      std::optional<std::pair<int, int>> best;
      Ratio best_eft = 0;
      for (int d : available) {
        Ratio eft = component_time(c, platform_.device(d).type);  // + residual 0: d is idle
        if (!best || eft < best_eft) {
          best = std::make_pair(c, d);
          best_eft = eft;
        }
      }
      return best;
    }
  }
  return std::nullopt;
}

std::optional<std::pair<int, int>> Scheduler::select_heft_waits(const Ratio& now) const {
  if (frontier_.empty()) return std::nullopt;
  int c = *frontier_.begin();
  for (int f : frontier_)
    if (comp_rank_[size_t(c)] < comp_rank_[size_t(f)]) c = f;  // max rank, ties lower id
  std::optional<int> best;
  Ratio best_eft = 0;
  for (const auto& dev : platform_.devices) {  // ascending id: ties go to the lower id
    Ratio residual = 0;
    if (!available_.count(dev.id))
      for (const auto& [comp, live] : live_)
        if (live.device == dev.id && now < live.release) residual = live.release - now;
    const Ratio eft = residual + component_time(c, dev.type);
    if (!best || eft < best_eft) {
      best = dev.id;
      best_eft = eft;
    }
  }
  if (!available_.count(*best)) return std::nullopt;  // the best device is busy: wait for it
  return std::make_pair(c, *best);
}

void Scheduler::mark_finished(int kernel, ScheduleResult& out) {
  if (finished_.insert(kernel).second) out.kernel_finish_order.push_back(kernel);
}

void Scheduler::enqueue_ready(std::set<int>& frontier) {
  for (size_t c = 0; c < comps_.size(); ++c) {
    if (state_[c] != State::waiting) continue;
    bool ok = std::all_of(cross_preds_[c].begin(), cross_preds_[c].end(),
                          [&](int k) { return finished_.count(k) > 0; });
    if (ok) {
      state_[c] = State::queued;
      frontier.insert(int(c));
    }
  }
}

void Scheduler::cb(const Completion& c, ScheduleResult& out) {
  auto it = live_.find(c.component);
  if (it == live_.end())
    fail(Errc::unknown_event, "component " + std::to_string(c.component) + " is not dispatched");
  Live& live = it->second;
  if (!live.q.callbacks.count(c.event))
    fail(Errc::unknown_event, "event " + std::to_string(c.event) + " of component " + std::to_string(c.component) +
                                  " has no callback");
  out.completions.push_back(c);
  live.done_events.insert(c.event);
  const TaskComponent& t = comps_[size_t(c.component)];
  const DeviceType dt = platform_.device(live.device).type;

  // update_status: END kernels finish on their marked events.
  for (int k : t.end) {
    if (finished_.count(k)) continue;
    bool any = false, all = true;
    for (int ev : live.q.end_marks) {
      const Command& cmd = live.q.command_of(ev);
      if (cmd.kernel != k) continue;
      if (dt == DeviceType::gpu && cmd.kind != CmdKind::read) continue;
      if (dt == DeviceType::cpu && cmd.kind != CmdKind::ndrange) continue;
      any = true;
      all = all && live.done_events.count(ev);
    }
    if (any && all) mark_finished(k, out);
  }
  // Component completion: every queue's terminal command has completed.
  auto terms = live.q.terminal_events();
  bool complete = std::all_of(terms.begin(), terms.end(), [&](int ev) { return live.done_events.count(ev) > 0; });
  if (complete) {
    for (int k : t.kernel_ids) mark_finished(k, out);
    state_[size_t(c.component)] = State::done;
    available_.insert(live.device);  // return_device
    live_.erase(it);
  }
  enqueue_ready(frontier_);  // get_ready_succ + update_task_queue
}

ScheduleResult Scheduler::run(Executor& ex) {
  ScheduleResult out;
  state_.assign(comps_.size(), State::waiting);
  finished_.clear();
  frontier_.clear();
  available_.clear();
  live_.clear();
  for (const auto& d : platform_.devices) available_.insert(d.id);
  enqueue_ready(frontier_);  // F <- ready_task_components(G)

  const size_t total = g_.kernels.size();
  while (finished_.size() < total) {
    while (!available_.empty() && !frontier_.empty()) {
      const bool waits = heft_waits_ && policy_ == Policy::heft;
      auto pick = waits ? select_heft_waits(ex.clock().value_or(Ratio(0))) : select(frontier_, available_);
      if (!pick) break;  // select blocks until a callback changes F or A
      auto [c, d] = *pick;
      const DeviceInfo& dev = platform_.device(d);
      if (!available_.count(d)) fail(Errc::device_busy, "device " + std::to_string(d));
      CommandQueueStructure q = setup_cq(comps_[size_t(c)], d, dev.type, dev.queues, g_, ec_);
      frontier_.erase(c);
      available_.erase(d);
      state_[size_t(c)] = State::dispatched;
      Live live;
      live.device = d;
      live.q = q;
      live.release = ex.clock().value_or(Ratio(0)) + component_time(c, dev.type);
      live_.emplace(c, std::move(live));
      out.dispatches.push_back({c, d});
      out.structures.push_back(q);
      ex.dispatch(comps_[size_t(c)], q);
    }
    if (finished_.size() >= total) break;
    if (live_.empty())
      fail(Errc::deadlock, std::to_string(total - finished_.size()) +
                               " kernels unfinished and no dispatched component can make progress");
    cb(ex.wait_next(), out);  // sleep_till_cb_update
  }
  return out;
}

ScheduleResult run_schedule(const DagSpec& g, const Platform& p, const Profiles& prof, Policy policy, Executor& ex,
                            bool heft_waits) {
  Scheduler s(g, p, prof, policy);
  s.set_heft_waits(heft_waits);
  return s.run(ex);
}

void PlanExecutor::dispatch(const TaskComponent& t, const CommandQueueStructure& q) {
  for (int ev : q.callbacks) pending_.push_back({t.id, ev});
}

Completion PlanExecutor::wait_next() {
  if (pending_.empty()) fail(Errc::deadlock, "no outstanding events");
  Completion c = pending_.front();
  pending_.pop_front();
  return c;
}

void ReplayExecutor::dispatch(const TaskComponent& t, const CommandQueueStructure& q) {
  (void)q;
  dispatched_.insert(t.id);
}

Completion ReplayExecutor::wait_next() {
  if (next_ >= log_.size()) fail(Errc::deadlock, "replay log exhausted");
  Completion c = log_[next_++];
  if (!dispatched_.count(c.component))
    fail(Errc::unknown_event, "replayed completion for undispatched component " + std::to_string(c.component));
  return c;
}

}  // namespace hetsim
