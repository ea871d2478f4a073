"""Command-line entry point (SPEC.md `cli` module): validate / simulate / run /
compare / sweep over the host API, the platform simulator and the B200 engine.

  python -m paper_2009_07482_b200 validate --spec dag.json [--params N=256 ...]
  python -m paper_2009_07482_b200 simulate --spec dag.json --profiles prof.json [--policy clustering]
                                           [--gantt text|svg|none] [--callback-delay MS] [--cpu-devices 1]
                                           [--heft-waits]
  python -m paper_2009_07482_b200 run      --spec dag.json [--policy P] [--mode graph|dynamic] [--instances N]
                                           [--gantt text|svg|none] [--out DIR]          (B200)
  python -m paper_2009_07482_b200 compare  --spec dag.json --profiles prof.json --policies clustering,eager,heft
  python -m paper_2009_07482_b200 sweep    --heads H [--beta 256] [--qgpu 1-5] [--qcpu 1-5] [--hcpu 0-H]
                                           [--profiles prof.json | --measure] [--out DIR]

Exit codes (SPEC.md cli invariants; proj/src/errors.cpp:33-45): 0 success, 1 runtime
error (deadlock, device error, ...), 2 input error (malformed spec, usage).
`simulate` / `compare` / `sweep --profiles` need no GPU. A profiles file is
{"devices": [{"device": 0, "type": "gpu", "kernel_times": {"<kernel id>": ms, ...},
"kernel_share": {...}, "copy_channels": 2, "bandwidth": bytes_per_ms,
"transfer_latency": ms}, ...]} (hs_query "simulate"); for `sweep` it is
{"gpu": {"gemm": ms, "transpose": ms, "softmax": ms}, "cpu": {...}, "share": {...}}.
"""
from __future__ import annotations

import argparse
import json
import pathlib
import sys
from fractions import Fraction

from . import _native, hetsim, reporting, sweep


class UsageError(ValueError):
    """Bad command-line usage (exit 2)."""


def _params(items):
    out = {}
    for it in items or []:
        k, _, v = it.partition("=")
        if not k or not v:
            raise UsageError(f"--params expects K=V, got {it!r}")
        out[k] = int(v) if v.lstrip("-").isdigit() else v
    return out


def _range(text, default):
    if text is None:
        return default
    if "-" in text:
        a, b = text.split("-", 1)
        return range(int(a), int(b) + 1)
    return [int(x) for x in text.split(",")]


def _frac(x) -> str:
    return str(Fraction(str(x)).limit_denominator(10**6)) if not isinstance(x, str) else x


def _profiles(path):
    doc = json.loads(pathlib.Path(path).read_text())
    devs = doc["devices"] if isinstance(doc, dict) and "devices" in doc else doc
    for d in devs:
        for key in ("kernel_times", "kernel_share"):
            if key in d:
                d[key] = {str(k): _frac(v) for k, v in d[key].items()}
        for key in ("bandwidth", "transfer_latency"):
            if key in d:
                d[key] = _frac(d[key])
    return devs


def _emit(out_dir, name, text):
    if out_dir:
        p = pathlib.Path(out_dir)
        p.mkdir(parents=True, exist_ok=True)
        (p / name).write_text(text)


def _sim(spec_text, params, profiles, policy, delay, cpu_devices, heft_waits=False):
    return _native.query({"op": "simulate", "spec": spec_text, "params": params, "policy": policy,
                          "cpu_devices": cpu_devices, "device_profiles": profiles,
                          "callback_delay": _frac(delay), "heft_waits": int(bool(heft_waits))})["simulate"]


def _float_trace(tr):
    return [{**r, "start": float(Fraction(r["start"])), "finish": float(Fraction(r["finish"]))} for r in tr]


def cmd_validate(a):
    text = pathlib.Path(a.spec).read_text()
    spec = hetsim.parse_spec(text, _params(a.params))
    an = hetsim.analyze(spec)
    # evaluates every size: unbound parameters surface here
    an["buffer_bytes"] = {f"{k}.{pos}": b for (k, pos), b in hetsim.buffer_bytes(spec).items()}
    print(json.dumps(an, indent=1))


def cmd_simulate(a):
    text = pathlib.Path(a.spec).read_text()
    s = _sim(text, _params(a.params), _profiles(a.profiles), a.policy, a.callback_delay, a.cpu_devices,
             a.heft_waits)
    tr = _float_trace(s["trace"])
    print(f"makespan_ms {s['makespan_ms']:.6f}")
    if a.gantt != "none":
        g = reporting.gantt(tr, a.gantt, quantum=a.quantum)
        print(g) if a.gantt == "text" else _emit(a.out, "gantt.svg", g)
    _emit(a.out, "trace.json", json.dumps(s["trace"], indent=1))


def cmd_compare(a):
    text = pathlib.Path(a.spec).read_text()
    policies = [p for p in a.policies.split(",") if p]
    if not policies:
        raise UsageError("--policies is empty")
    runs = []
    for pol in policies:
        s = _sim(text, _params(a.params), _profiles(a.profiles), pol, a.callback_delay, a.cpu_devices,
                 a.heft_waits)
        runs.append((pol, _float_trace(s["trace"])))
    csv = reporting.compare_csv(runs)
    print(csv, end="")
    _emit(a.out, "compare.csv", csv)


def cmd_run(a):
    import numpy as np

    from . import workloads
    from .engine import Engine
    text = pathlib.Path(a.spec).read_text()
    params = _params(a.params)
    arrays = workloads.generic_inputs(text, params, a.instances)
    outs = {(k, p): np.zeros((a.instances, e), np.float32) for k, p, e in workloads.isolated_outputs(text, params)}
    with Engine(text, params, policy=a.policy, mode=a.mode, batch=a.batch or a.instances, trace=True) as eng:
        for key, arr in arrays.items():
            eng.bind(*key, arr)
        for key, arr in outs.items():
            eng.bind(*key, arr)
        eng.run(0, a.instances)  # plan, capture, upload
        ns = eng.run(0, a.instances)
        tr = eng.trace()
    print(f"makespan_ms {ns / 1e6:.6f}  (instances {a.instances}, traced batch {reporting.makespan(tr):.6f} ms)")
    if a.gantt != "none":
        g = reporting.gantt(tr, a.gantt, quantum=a.quantum)
        print(g) if a.gantt == "text" else _emit(a.out, "gantt.svg", g)
    _emit(a.out, "trace.json", json.dumps(tr, indent=1))
    if a.out:
        for (k, p), arr in outs.items():
            np.save(pathlib.Path(a.out) / f"out_k{k}_p{p}.npy", arr)


def cmd_sweep(a):
    if a.measure:
        gpu_t, share = sweep.gpu_node_times(a.beta)
        cpu_t = sweep.cpu_node_times(a.beta)
    elif a.profiles:
        doc = json.loads(pathlib.Path(a.profiles).read_text())
        gpu_t, cpu_t, share = doc["gpu"], doc["cpu"], doc.get("share")
    else:
        raise UsageError("sweep needs --profiles FILE or --measure")
    hc = _range(a.hcpu, None)
    if hc is not None and any(h > a.heads or h < 0 for h in hc):
        raise UsageError(f"--hcpu must be within [0, {a.heads}]")
    t = sweep.sweep_clustering(a.heads, a.beta, gpu_t, cpu_t, share, q_gpu=_range(a.qgpu, range(1, 6)),
                               q_cpu=_range(a.qcpu, range(1, 6)), h_cpu=hc)
    csv = sweep.to_csv(t)
    print(csv, end="")
    print(f"best {sweep.label(t['best']['mc'])} {t['best']['makespan_ms']:.6f} ms; "
          f"best vs default <1,0,0>: {t['best_vs_default']:.3f}x" if t["best_vs_default"] else "")
    _emit(a.out, "sweep.csv", csv)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2009_07482_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)

    def common(p, profiles=False):
        p.add_argument("--spec", required=True)
        p.add_argument("--params", nargs="*", default=[])
        p.add_argument("--out")
        if profiles:
            p.add_argument("--profiles", required=True)
            p.add_argument("--callback-delay", type=float, default=0.0)
            p.add_argument("--cpu-devices", type=int, nargs="*", default=[])
            # SPEC.md:358 / :551: HEFT weighs busy devices by their release time
            p.add_argument("--heft-waits", action="store_true")

    p = sub.add_parser("validate")
    common(p)
    p = sub.add_parser("simulate")
    common(p, profiles=True)
    p.add_argument("--policy", choices=["clustering", "eager", "heft"], default="clustering")
    p.add_argument("--gantt", choices=["text", "svg", "none"], default="none")
    p.add_argument("--quantum", type=float, default=1.0)
    p = sub.add_parser("compare")
    common(p, profiles=True)
    p.add_argument("--policies", default="clustering,eager,heft")
    p = sub.add_parser("run")
    common(p)
    p.add_argument("--policy", choices=["clustering", "eager", "heft"], default="clustering")
    p.add_argument("--mode", choices=["graph", "dynamic"], default="graph")
    p.add_argument("--instances", type=int, default=1)
    p.add_argument("--batch", type=int, default=0)
    p.add_argument("--gantt", choices=["text", "svg", "none"], default="none")
    p.add_argument("--quantum", type=float, default=0.01)
    p = sub.add_parser("sweep")
    p.add_argument("--heads", type=int, required=True)
    p.add_argument("--beta", type=int, default=256)
    p.add_argument("--qgpu")
    p.add_argument("--qcpu")
    p.add_argument("--hcpu")
    p.add_argument("--profiles")
    p.add_argument("--measure", action="store_true")
    p.add_argument("--out")
    a = ap.parse_args(argv)
    try:
        {"validate": cmd_validate, "simulate": cmd_simulate, "compare": cmd_compare, "run": cmd_run,
         "sweep": cmd_sweep}[a.cmd](a)
    except _native.HetsimError as e:
        print(str(e), file=sys.stderr)
        return e.exit_code if e.exit_code is not None else 1
    except UsageError as e:
        print(f"usage error: {e}", file=sys.stderr)
        return 2
    except (OSError, json.JSONDecodeError, KeyError, ValueError) as e:
        print(f"InputError: {e}", file=sys.stderr)
        return 2
    return 0


if __name__ == "__main__":
    sys.exit(main())
