"""C1-C3 makespans: cluster split-K (default lib) vs red.add split-K (HETSIM_LIB=variants/lib_nocs.so),
and C3 with whole-head launches (fuse 3) vs grouped QKV + attn_head (fuse 2). usage: python profiles/r2_c3_fuse.py"""
import json
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402

for cfg, kw in (("C1", {}), ("C2", {}), ("C3", {"devices": 9}), ("C3", {"devices": 9, "fuse": 2})):
    r = bench.config_makespan(cfg, check=True, **kw)
    print(cfg, json.dumps(kw), json.dumps({"makespan_ms": r["makespan_ms"], "min_ms": r["makespan_min_ms"],
                                           "launches": r["launches"], "err": r["normwise_err_vs_cpu_oracle"]}))
