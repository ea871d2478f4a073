"""Expt. 1 of the paper on B200: clustering sweep over architecture mapping
configurations mc = <q_gpu, q_cpu, h_cpu> (SPEC.md `sweep_clustering`).

For a transformer-head DAG of H heads (`workloads.head_dag`, all
matrices beta x beta), every mc runs Alg. 1's clustering policy: h_cpu heads are
mapped to the CPU device (q_cpu queues), the others to the GPU (q_gpu queues).
mc = (1, 0, 0) is the paper's default coarse-grained scheme. Two columns:

  simulated  platform_sim (hs_query "simulate") fed with kernel times
             measured on this machine: GPU times of each node on the B200 (engine
             trace, one launch per ndrange), CPU times of numpy's fp32 kernels on the
             host. Covers the whole grid, CPU heads included.
  measured   the same DAG on the B200 through the engine (graph mode, one launch per
             ndrange = the paper's execution model; all heads on the GPU, so only
             configurations with h_cpu = 0). The CPU never executes a node on the
             product path (north_star: no CPU fallback).

The grid is the cartesian product of the valid configurations, each simulated
once (SPEC.md sweep invariants); q_cpu >= 1 whenever h_cpu > 0, q_cpu = 0 otherwise.
"""
from __future__ import annotations

import json
from fractions import Fraction

from . import _native, workloads

GPU_DEVICE, CPU_DEVICE = 0, 1


def head_spec(heads: int, beta: int, q_gpu: int, q_cpu: int, h_cpu: int) -> tuple[str, dict]:
    """head_dag with the first h_cpu heads on the CPU device (its own cq entry)."""
    if not 0 <= h_cpu <= heads:
        raise ValueError(f"h_cpu must be in [0, {heads}]")
    if q_gpu < 1 and h_cpu < heads:
        raise ValueError("GPU heads need q_gpu >= 1")
    if h_cpu > 0 and q_cpu < 1:
        raise ValueError("CPU heads need q_cpu >= 1")
    text, params = workloads.head_dag(heads=heads, beta=beta, queues=max(q_gpu, 1))
    doc = json.loads(text)
    per_head = len(doc["kernels"]) // heads
    for k in doc["kernels"]:
        if k["id"] // per_head < h_cpu:
            k["dev"] = "cpu"
    cq = []
    if h_cpu < heads:
        cq.append({"device": GPU_DEVICE, "queues": q_gpu})
    if h_cpu > 0:
        cq.append({"device": CPU_DEVICE, "queues": q_cpu})
    doc["cq"] = cq
    return json.dumps(doc, indent=1), params


def configurations(heads: int, q_gpu=range(1, 6), q_cpu=range(1, 6), h_cpu=None):
    """Valid mc = (q_gpu, q_cpu, h_cpu): q_cpu = 0 iff h_cpu = 0; q_gpu only matters
    while a head is left on the GPU (h_cpu = H uses q_gpu = 0)."""
    h_range = range(0, heads + 1) if h_cpu is None else h_cpu
    out = []
    for h in h_range:
        gq = [0] if h == heads else list(q_gpu)
        cq = [0] if h == 0 else list(q_cpu)
        for g in gq:
            for c in cq:
                out.append((g, c, h))
    return out


def _frac(ms: float) -> str:
    return str(Fraction(round(ms * 1e3), 1000))  # microsecond resolution keeps the rationals small


def simulate(heads: int, beta: int, mc, gpu_times: dict, cpu_times: dict, gpu_share: dict | None = None,
             callback_delay_ms: float = 0.0, bandwidth_Bpms: float | None = None, latency_ms: float = 0.0) -> dict:
    """platform_sim makespan of one configuration. gpu_times / cpu_times: node role
    ('gemm', 'transpose', 'softmax') -> ms; gpu_share: role -> fraction of the GPU one
    such kernel occupies (processor sharing beyond 1)."""
    q_gpu, q_cpu, h_cpu = mc
    text, params = head_spec(heads, beta, q_gpu, q_cpu, h_cpu)
    doc = json.loads(text)
    role = {k["id"]: ("gemm" if k["name"].startswith("gemm") else k["name"]) for k in doc["kernels"]}
    profiles = []
    # transfers: device-resident by default (the measured column copies inputs D2D)
    chan = {"copy_channels": 2, "bandwidth": str(int(round(bandwidth_Bpms))) if bandwidth_Bpms else "1000000000000",
            "transfer_latency": _frac(latency_ms)}
    if h_cpu < heads:
        prof = {"device": GPU_DEVICE, "type": "gpu", "kernel_times": {str(k): _frac(gpu_times[r]) for k, r in role.items()}}
        if gpu_share:
            prof["kernel_share"] = {str(k): str(Fraction(gpu_share[r]).limit_denominator(1000)) for k, r in role.items()}
        profiles.append({**prof, **chan})
    if h_cpu > 0:
        profiles.append({"device": CPU_DEVICE, "type": "cpu", "copy_channels": 1, "bandwidth": "1000000000000",
                         "transfer_latency": "0",
                         "kernel_times": {str(k): _frac(cpu_times[r]) for k, r in role.items()}})
    s = _native.query({"op": "simulate", "spec": text, "params": params, "policy": "clustering",
                       "cpu_devices": [CPU_DEVICE] if h_cpu > 0 else [], "device_profiles": profiles,
                       "callback_delay": _frac(callback_delay_ms)})["simulate"]
    return {"mc": list(mc), "makespan_ms": s["makespan_ms"], "dispatches": s["dispatches"]}


def sweep_clustering(heads: int, beta: int, gpu_times: dict, cpu_times: dict, gpu_share: dict | None = None,
                     q_gpu=range(1, 6), q_cpu=range(1, 6), h_cpu=None, **sim_kw) -> dict:
    """The simulated sweep table plus the best-vs-default (mc = (1,0,0)) speedup."""
    rows = [simulate(heads, beta, mc, gpu_times, cpu_times, gpu_share, **sim_kw)
            for mc in configurations(heads, q_gpu, q_cpu, h_cpu)]
    default = next((r for r in rows if r["mc"] == [1, 0, 0]), None)
    best = min(rows, key=lambda r: r["makespan_ms"])
    return {"heads": heads, "beta": beta, "rows": rows, "best": best,
            "default": default, "best_vs_default": (default["makespan_ms"] / best["makespan_ms"]) if default else None}


def label(mc) -> str:
    """Fig. 9-style label of a configuration."""
    return f"<{mc[0]},{mc[1]},{mc[2]}>"


def to_csv(table: dict) -> str:
    lines = ["heads,beta,q_gpu,q_cpu,h_cpu,label,makespan_ms,best"]
    for r in table["rows"]:
        g, c, h = r["mc"]
        lines.append(f"{table['heads']},{table['beta']},{g},{c},{h},{label(r['mc'])},{r['makespan_ms']:.6f},"
                     f"{int(r is table['best'])}")
    return "\n".join(lines) + "\n"


# ----------------------------------------------------------------------------- profiles measured here

def gpu_node_times(beta: int = 256, reps: int = 3) -> tuple[dict, dict]:
    """Standalone time of each node role of the head DAG on the B200: one head,
    one queue, one launch per ndrange, every command timed with CUDA events
    (engine trace). Returns (role -> ms, role -> share of the GPU = CTAs / SMs)."""
    import numpy as np
    import torch

    from .engine import Engine
    text, params = workloads.head_dag(heads=1, beta=beta, queues=1)
    arrays = workloads.generic_inputs(text, params, 1)
    outs = {(k, p): np.zeros((1, e), np.float32) for k, p, e in workloads.isolated_outputs(text, params)}
    best: dict = {}
    with Engine(text, params, batch=1, mode="graph", fuse=0, trace=True) as eng:
        for key, a in arrays.items():
            eng.bind(*key, a)
        for key, a in outs.items():
            eng.bind(*key, a)
        doc = json.loads(text)
        role = {k["id"]: ("gemm" if k["name"].startswith("gemm") else k["name"]) for k in doc["kernels"]}
        for _ in range(reps + 1):
            eng.run(0, 1)
            for r in eng.trace():
                if r["kind"] == "ndrange":
                    t = r["finish"] - r["start"]
                    ro = role[r["kernel"]]
                    best[ro] = min(best.get(ro, t), t)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    tiles = (-(-beta // 128)) ** 2  # 128 x 128 output tiles of a beta x beta GEMM
    share = {"gemm": min(1.0, tiles / sms), "transpose": min(1.0, beta * beta / 1024 / 4 / sms),
             "softmax": min(1.0, beta / 8 / sms)}
    return best, share


def cpu_node_times(beta: int = 256, reps: int = 5) -> dict:
    """Time of each node role on this host's CPU (the CPU device of the simulated
    platform), with numpy's fp32 kernels: BLAS sgemm, a strided transpose copy and a
    row softmax. Best of `reps`."""
    import time

    import numpy as np
    a = np.random.default_rng(0).standard_normal((beta, beta)).astype(np.float32)

    def softmax(x):
        e = np.exp(x - x.max(axis=1, keepdims=True))
        return e / e.sum(axis=1, keepdims=True)

    cases = {"gemm": lambda: a @ a, "transpose": lambda: np.ascontiguousarray(a.T), "softmax": lambda: softmax(a)}
    res = {}
    for ro, fn in cases.items():
        fn()
        t = []
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            t.append((time.perf_counter() - t0) * 1e3)
        res[ro] = min(t)
    return res


def measured_gpu_makespan(heads: int, beta: int, q_gpu: int, reps: int = 10, devices: int = 1) -> float:
    """The head DAG (all heads on the GPU) on the B200: graph mode, one launch per
    ndrange, device-resident inputs; median engine makespan in ms."""
    import statistics

    import torch

    from .engine import Engine
    text, params = workloads.head_dag(heads=heads, beta=beta, queues=q_gpu)
    if devices > 1:
        doc = json.loads(text)
        doc["cq"] = workloads.cq_list(devices, q_gpu)
        text = json.dumps(doc, indent=1)
    arrays = workloads.generic_inputs(text, params, 1)
    dev = {k: torch.from_numpy(a).cuda() for k, a in arrays.items()}
    outs = {(k, p): torch.zeros(1, e, device="cuda") for k, p, e in workloads.isolated_outputs(text, params)}
    torch.cuda.synchronize()
    with Engine(text, params, batch=1, mode="graph", fuse=0) as eng:
        for key, t in dev.items():
            eng.bind(*key, t)
        for key, t in outs.items():
            eng.bind(*key, t)
        for _ in range(3):
            eng.run(0, 1)
        ns = [eng.run(0, 1) for _ in range(reps)]
    return statistics.median(ns) / 1e6
