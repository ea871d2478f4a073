"""Per-node roofline and the whole-DAG makespan bound T* (SURVEY.md §8d).

    t_n  = max(F_n / P, bytes_n / B)                      per node, one instance
    T*   = max(critical path over t_n,                    (latency bound of one instance)
               n * sum F_n / P,                           (compute over n instances)
               (resident bytes + n * instance I/O) / B)   (compulsory HBM traffic)

F_n and bytes_n are ALGORITHMIC work (DESIGN.md §5 "algorithmic work"), read off
the spec's kernel names and var-args with the operator conventions of DESIGN.md
§4. P is the fp32-accurate GEMM peak (dense TF32 / 3 for 3xTF32), B the measured
HBM bandwidth. Host-side only; no device code.
"""
from __future__ import annotations

import json

from .workloads import _eval


def _var_args(k, params):
    return [_eval(v["value"], params) for v in sorted(k.get("varArguments", []), key=lambda v: v["pos"])]


def _sizes(k, params, field):
    return [_eval(b["size"], params) for b in sorted(k.get(field, []), key=lambda b: b["pos"])]


def node_work(k: dict, params: dict) -> tuple[float, float]:
    """(flops, bytes) of one instance of spec kernel `k` (DESIGN.md §4 conventions)."""
    name = k["name"]
    va = _var_args(k, params)
    if name in ("gemm", "gemm_nt", "gemm_relu"):
        m, n, kk = va[:3]
        return 2.0 * m * n * kk, 4.0 * (m * kk + kk * n + m * n)
    if name == "attn_head":
        s, dk, dw = va[:3]
        return 2.0 * s * s * dk * 2 + 2.0 * s * dk * dw, 4.0 * (3 * s * dk + dk * dw + s * dw)
    if name == "add_layernorm":
        r, c = va[:2]
        return 8.0 * r * c, 4.0 * 3 * r * c + 8.0 * c
    # elementwise / softmax / transpose / concat / add / scale: one pass, in + out
    ins, outs = _sizes(k, params, "inputBuffers"), _sizes(k, params, "outputBuffers")
    return 0.0, 4.0 * (sum(ins) + sum(outs))


def dag_bound(spec_text: str, params: dict, n_instances: int, peak_tflops: float, hbm_gbs: float,
              shared_inputs=(), io_bytes: float | None = None) -> dict:
    """T* for n independent instances of the DAG on one GPU. `shared_inputs` lists the
    (kernel, pos) inputs that are resident weights (read once per GPU, not per instance).
    `io_bytes` overrides the per-instance input+output bytes when several isolated
    inputs are bound to one host buffer (the encoder's X feeds 25 kernels)."""
    doc = json.loads(spec_text)
    P, B = peak_tflops * 1e12, hbm_gbs * 1e9
    kernels = {k["id"]: k for k in doc["kernels"]}
    work = {kid: node_work(k, params) for kid, k in kernels.items()}
    t = {kid: max(f / P, b / B) for kid, (f, b) in work.items()}
    succ = {kid: [] for kid in kernels}
    indeg = {kid: 0 for kid in kernels}
    for s, _, d, _ in doc.get("depends", []):
        succ[s].append(d)
        indeg[d] += 1
    # longest path (Kahn order)
    order, frontier = [], sorted(k for k, v in indeg.items() if v == 0)
    deg = dict(indeg)
    while frontier:
        u = frontier.pop(0)
        order.append(u)
        for v in succ[u]:
            deg[v] -= 1
            if deg[v] == 0:
                frontier.append(v)
    finish = {}
    start = {kid: 0.0 for kid in kernels}
    for u in order:
        finish[u] = start[u] + t[u]
        for v in succ[u]:
            start[v] = max(start[v], finish[u])
    cp = max(finish.values(), default=0.0)
    flops = sum(f for f, _ in work.values())
    fed = {(e[2], e[3]) for e in doc.get("depends", [])}
    feeding = {(e[0], e[1]) for e in doc.get("depends", [])}
    shared = {tuple(x) for x in shared_inputs}
    resident, io = 0.0, 0.0
    for k in doc["kernels"]:
        for b in k.get("inputBuffers", []) + k.get("ioBuffers", []):
            key = (k["id"], b["pos"])
            if key in fed:
                continue
            nbytes = 4.0 * _eval(b["size"], params)
            if key in shared:
                resident += nbytes
            else:
                io += nbytes
        for b in k.get("outputBuffers", []) + k.get("ioBuffers", []):
            if (k["id"], b["pos"]) not in feeding:
                io += 4.0 * _eval(b["size"], params)
    if io_bytes is not None:
        io = float(io_bytes)
    compulsory = resident + n_instances * io
    t_compute = n_instances * flops / P
    t_hbm = compulsory / B
    t_star = max(cp, t_compute, t_hbm)
    return {"critical_path_ms": cp * 1e3, "compute_ms": t_compute * 1e3, "hbm_ms": t_hbm * 1e3,
            "t_star_ms": t_star * 1e3, "flop_per_instance": flops, "instances": n_instances,
            "bound": "critical_path" if t_star == cp else ("tensor" if t_star == t_compute else "hbm")}
