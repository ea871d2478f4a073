"""Makespans of the latency configs C1-C4 (bench.config_makespan: graph mode, device-
resident, median of 20 runs), for an A/B of programmatic dependent launch:
HS_PDL=0 python profiles/pdl_probe.py  vs  python profiles/pdl_probe.py"""
import json
import os
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402

out = {"pdl": os.environ.get("HS_PDL", "1") != "0"}
for cfg, kw in (("C1", {}), ("C2", {}), ("C3", {"devices": 9}), ("C4", {"devices": 9})):
    r = bench.config_makespan(cfg, check=False, **kw)
    out[cfg] = {"makespan_ms": r["makespan_ms"], "min_ms": r["makespan_min_ms"], "t_star_ms": r["t_star_ms"],
                "launches": r["launches"]}
print(json.dumps(out))
