"""Latency configs C1-C4 (bench.config_makespan: graph mode, device-resident, median of
20 runs) with and without the engine's whole-run graph (run_graph: copies + plan in one
graph, one host submission per run), plus the host wall time of one run() call.
usage: python profiles/run_graph_probe.py"""
import json
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402

out = {}
for rg in (False, True):
    for cfg, kw in (("C1", {}), ("C2", {}), ("C3", {"devices": 9}), ("C4", {"devices": 9})):
        r = bench.config_makespan(cfg, check=(cfg != "C4"), run_graph=rg, **kw)
        out[f"{cfg}_run_graph{int(rg)}"] = {"makespan_ms": r["makespan_ms"], "min_ms": r["makespan_min_ms"],
                                           "normwise_vs_oracle": r.get("normwise_err_vs_cpu_oracle")}
for k, v in out.items():
    print(k, json.dumps(v))
