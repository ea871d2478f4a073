"""TEST INFRASTRUCTURE ONLY — CPU restatement of platform_sim,
used by tests/ as the checker for the product's C++ simulator
(csrc/sched/platform_sim.cpp). The reference specifies this module in prose
only (no code); parity is pinned by SPEC's worked examples
and by product == restatement on random DAGs, policies and profiles.

Rules restated (SPEC.md line refs):
  :389  runnable = queue predecessor done, E_Q predecessors done, resource free
  :396  transfer_time = latency + bytes / bandwidth on a GPU, 0 on a CPU
  :404  processor sharing: sigma = sum of shares of running ndranges on a
        device; each runs at rate 1 if sigma <= 1 else 1 / sigma
  :412  channel = earliest free (ties: lower id), FIFO per channel
  :433  equal completion times complete in (device, queue, position) order
Callback-marked completions reach the scheduler `callback_delay` later;
completions at a time are processed before callbacks delivered at that time.
B200 extension: issuing a component occupies the host for `dispatch_cost`, one
component at a time; its commands start no earlier than that.
"""
from __future__ import annotations

from fractions import Fraction

from .oracle import OracleError, Spec, schedule


def F(x) -> Fraction:
    return x if isinstance(x, Fraction) else Fraction(str(x))


def transfer_time(nbytes: int, prof: dict) -> Fraction:
    if prof["type"] == "cpu":
        return Fraction(0)
    return F(prof.get("transfer_latency", 0)) + Fraction(nbytes) / F(prof.get("bandwidth", 1))


class Sim:
    def __init__(self, profiles: list[dict], callback_delay=0, dispatch_cost=0):
        self.prof = {p["device"]: p for p in profiles}
        self.delay = F(callback_delay)
        self.cost = F(dispatch_cost)
        self.host_free = Fraction(0)
        self.t = Fraction(0)
        self.cmds = []        # dicts
        self.free = {d: [Fraction(0)] * max(1, int(p.get("copy_channels", 2))) for d, p in self.prof.items()}
        self.deliver = []     # (time, seq, (c, ev))
        self.trace = []

    # -- executor interface used by oracle.schedule
    def dispatch(self, comp, device, q):
        base = len(self.cmds)
        self.host_free = max(self.t, self.host_free) + self.cost  # one component at a time on the host
        ev_index = {}
        for qi, evs in enumerate(q["_queues"]):
            for pos, ev in enumerate(evs):
                c = q["commands"][ev]
                ev_index[ev] = len(self.cmds)
                self.cmds.append({"comp": comp, "ev": ev, "device": device, "queue": qi, "pos": pos,
                                  "kind": c["kind"], "kernel": c["kernel"], "label": c["label"],
                                  "bytes": c.get("bytes", 0), "callback": ev in q["_callbacks"],
                                  "prev": ev_index[evs[pos - 1]] if pos else None, "preds": [],
                                  "st": "pending", "channel": -1, "ready_at": self.host_free})
        for a, b in q["_deps"]:
            self.cmds[ev_index[b]]["preds"].append(ev_index[a])
        assert base <= len(self.cmds)

    def _key(self, c):
        return (c["device"], c["queue"], c["pos"], c["comp"])

    def _rate(self, device):
        shares = self.prof[device].get("kernel_share", {})
        sigma = sum((F(shares.get(str(c["kernel"]), shares.get(c["kernel"], 1))) for c in self.cmds
                     if c["st"] == "running" and c["kind"] == "ndrange" and c["device"] == device), Fraction(0))
        return Fraction(1) if sigma <= 1 else 1 / sigma

    def _start(self):
        for c in sorted((c for c in self.cmds if c["st"] == "pending"), key=self._key):
            if self.t < c["ready_at"]:
                continue
            if c["prev"] is not None and self.cmds[c["prev"]]["st"] != "done":
                continue
            if any(self.cmds[p]["st"] != "done" for p in c["preds"]):
                continue
            p = self.prof[c["device"]]
            c["st"] = "running"
            if c["kind"] == "ndrange":
                times = p["kernel_times"]
                key = str(c["kernel"]) if str(c["kernel"]) in times else c["kernel"]
                if key not in times:
                    raise OracleError("MissingProfileEntry")
                c["start"], c["left"] = self.t, F(times[key])
            elif p["type"] == "cpu":
                c["start"] = c["finish"] = self.t
            else:
                free = self.free[c["device"]]
                ch = min(range(len(free)), key=lambda i: (free[i], i))
                c["channel"] = ch
                c["start"] = max(self.t, free[ch])
                c["finish"] = c["start"] + transfer_time(c["bytes"], p)
                free[ch] = c["finish"]

    def _advance(self, t):
        if t == self.t:
            return
        rates = {}
        for c in self.cmds:
            if c["st"] == "running" and c["kind"] == "ndrange":
                if c["device"] not in rates:
                    rates[c["device"]] = self._rate(c["device"])
                c["left"] -= rates[c["device"]] * (t - self.t)
        self.t = t

    def wait_next(self):
        while True:
            self._start()
            cand = []
            for i, c in enumerate(self.cmds):
                if c["st"] != "running":
                    continue
                f = self.t + c["left"] / self._rate(c["device"]) if c["kind"] == "ndrange" else c["finish"]
                cand.append((f, self._key(c), i))
            nxt = min(cand) if cand else None
            rel = min((c["ready_at"] for c in self.cmds if c["st"] == "pending" and self.t < c["ready_at"]),
                      default=None)
            if rel is not None and (nxt is None or rel < nxt[0]) and (not self.deliver or rel <= min(self.deliver)[0]):
                self._advance(rel)
                continue
            if self.deliver:
                d = min(self.deliver)
                if nxt is None or d[0] < nxt[0]:
                    self.deliver.remove(d)
                    self._advance(max(self.t, d[0]))
                    return d[2]
            if nxt is None:
                if any(c["st"] == "pending" for c in self.cmds):
                    raise OracleError("SimDeadlock")
                raise OracleError("Deadlock")
            f, _, i = nxt
            self._advance(f)
            c = self.cmds[i]
            c["st"], c["finish"], c["left"] = "done", self.t, Fraction(0)
            self.trace.append({"event": len(self.trace), "kind": c["kind"], "label": c["label"],
                               "kernel": c["kernel"], "component": c["comp"], "cmd_event": c["ev"],
                               "device": c["device"], "queue": c["queue"], "channel": c["channel"],
                               "start": c["start"], "finish": c["finish"]})
            if c["callback"]:
                self.deliver.append((self.t + self.delay, len(self.trace), (c["comp"], c["ev"])))

    def now(self):
        return self.t

    def makespan(self):
        if not self.trace:
            raise OracleError("EmptyTrace")
        return max(e["finish"] for e in self.trace) - min(e["start"] for e in self.trace)


def simulate(spec_text, params, profiles, policy="clustering", cpu_devices=(), callback_delay=0, heft_waits=False,
             dispatch_cost=0):
    """Alg. 1 (oracle.schedule) over the restated simulator. profiles: list of
    {"device", "type", "kernel_times", "kernel_share", "copy_channels", "bandwidth",
    "transfer_latency"}; the scheduler's per-type kernel times come from the first
    profile of each device type (as the product does)."""
    spec = Spec(spec_text, params)
    times = {}
    for p in profiles:
        per = times.setdefault(p["type"], {})
        for k, v in p["kernel_times"].items():
            per.setdefault(int(k), F(v))
    sim = Sim(profiles, callback_delay, dispatch_cost)
    sched = schedule(spec, policy=policy, times=times or None, cpu_devices=cpu_devices, executor=sim,
                     heft_waits=heft_waits)
    return {"schedule": sched, "trace": sim.trace, "makespan": sim.makespan()}
