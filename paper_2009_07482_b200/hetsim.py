"""Python mirror of the reference's C++ API (namespace ``hetsim``).

Same operation names and meaning as proj/include/hetsim/*.hpp, answered by the
native library through ``hs_query``. Errors surface as ``HetsimError`` with the
reference's Errc name (``MalformedSpec``, ``CycleDetected``, ...) and exit code
(2 for input errors, 1 for runtime errors; proj/src/errors.cpp:33-45).
"""
from __future__ import annotations

from dataclasses import dataclass, field

from ._native import HetsimError, query

__all__ = [
    "HetsimError", "DagSpec", "TaskComponent", "parse_spec", "serialize", "eval_expr", "eval_positive",
    "validate_expr", "derive_components", "classify_edges", "ready_components", "bottom_level_ranks",
    "setup_cq", "run_schedule", "buffer_bytes", "ratio",
]


@dataclass
class DagSpec:
    """A validated spec (canonical text + bindings), cf. spec_model.hpp DagSpec."""

    text: str
    params: dict = field(default_factory=dict)

    def _req(self, op: str, **kw) -> dict:
        return query({"op": op, "spec": self.text, "params": self.params, **kw})


@dataclass
class TaskComponent:
    id: int
    kernel_ids: list
    dev_pref: str
    front: set
    end: set
    interior: set


def parse_spec(text: str, params: dict | None = None) -> DagSpec:
    """parse_spec (spec_model.cpp:211): raises HetsimError on invalid documents."""
    params = dict(params or {})
    out = query({"op": "parse", "spec": text, "params": params})
    return DagSpec(out["serialized"], params)


def serialize(spec: DagSpec) -> str:
    return spec._req("parse")["serialized"]


def eval_expr(expr: str, params: dict | None = None) -> int:
    return query({"op": "expr", "expr": expr, "params": dict(params or {})})["value"]


def eval_positive(expr: str, params: dict | None = None) -> int:
    return query({"op": "expr", "expr": expr, "params": dict(params or {}), "mode": "positive"})["value"]


def validate_expr(expr: str) -> None:
    query({"op": "expr", "expr": expr, "mode": "validate"})


def ratio(a: str, b: str | None = None) -> dict:
    req = {"op": "ratio", "a": a}
    if b is not None:
        req["b"] = b
    return query(req)


def analyze(spec: DagSpec) -> dict:
    return spec._req("analyze")["analysis"]


def derive_components(spec: DagSpec) -> list[TaskComponent]:
    return [
        TaskComponent(c["id"], c["kernels"], c["dev_pref"], set(c["front"]), set(c["end"]), set(c["interior"]))
        for c in analyze(spec)["components"]
    ]


def classify_edges(spec: DagSpec) -> dict:
    a = analyze(spec)
    return {
        "edge_kind": a["edge_kind"],
        "write_class": {(k, p): c for k, p, c in a["write_class"]},
        "read_class": {(k, p): c for k, p, c in a["read_class"]},
    }


def ready_components(spec: DagSpec, finished) -> list[int]:
    return spec._req("ready", finished=sorted(finished))["ready"]


def bottom_level_ranks(spec: DagSpec, times: dict) -> tuple[dict, list]:
    out = spec._req("ranks", times={str(k): str(v) for k, v in times.items()})
    return {int(k): v for k, v in out["ranks"].items()}, out["component_ranks"]


def buffer_bytes(spec: DagSpec) -> dict:
    return {(k, p): b for k, p, b in spec._req("bytes")["bytes"]}


def setup_cq(spec: DagSpec, component: int, device: int = 0, device_type: str = "gpu", queues: int = 1) -> dict:
    """setup_cq (cq_builder.hpp:75): returns the to_debug_json() document."""
    return spec._req("setup_cq", component=component, device=device, device_type=device_type, queues=queues)["cq"]


def run_schedule(spec: DagSpec, policy: str = "clustering", times: dict | None = None, cpu_devices=(),
                 replay: list | None = None) -> dict:
    """Alg. 1 against the deterministic plan model, or replaying a completion log."""
    req = {"policy": policy, "cpu_devices": list(cpu_devices)}
    if times:
        req["times"] = {dev: {str(k): str(v) for k, v in per.items()} for dev, per in times.items()}
    if replay is not None:
        req["replay"] = [list(x) for x in replay]
    return spec._req("schedule", **req)["schedule"]
