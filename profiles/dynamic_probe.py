"""Dynamic mode (Alg. 1 literally: host callbacks -> scheduler -> dispatch) without
tracing: run time and the host-side split (dispatch vs waiting for callbacks).
usage: python profiles/dynamic_probe.py [out.json]"""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2009_07482_b200 import workloads  # noqa: E402
from paper_2009_07482_b200.engine import Engine  # noqa: E402

rows = []
for layers, batch, devices, policy in ((1, 1, 1, "clustering"), (1, 1, 9, "clustering"), (6, 64, 9, "clustering"),
                                       (6, 64, 9, "eager"), (6, 64, 9, "heft")):
    text, params, meta = workloads.encoder(layers=layers, devices=devices)
    x = workloads.encoder_inputs(meta, params, batch).reshape(batch, -1)
    out = np.zeros((batch, params["S"] * params["D"]), np.float32)
    res = {}
    for mode in ("dynamic", "dynamic_fused", "graph"):
        kw = {"dynamic_fuse": True} if mode == "dynamic_fused" else {}
        with Engine(text, params, mode="graph" if mode == "graph" else "dynamic", policy=policy, batch=batch,
                    **kw) as eng:
            for i in meta["x_inputs"]:
                eng.bind(i["kernel"], i["pos"], x)
            for k, w in workloads.encoder_weights(meta).items():
                eng.bind(*k, w.reshape(-1), shared=True)
            eng.bind(meta["output"]["kernel"], meta["output"]["pos"], out)
            eng.run(0, batch)
            before = eng.info("stats")
            ns = [eng.run(0, batch) for _ in range(3)]
            st = eng.info("stats")
        res[mode] = min(ns) / 1e6
        if mode != "graph":
            d = st["host_dispatches"] - before["host_dispatches"]
            res[mode + "_dispatch_us"] = (st["host_dispatch_us"] - before["host_dispatch_us"]) / max(d, 1)
        if mode == "dynamic":
            d = st["host_dispatches"] - before["host_dispatches"]
            res["dispatch_us_per_component"] = (st["host_dispatch_us"] - before["host_dispatch_us"]) / max(d, 1)
            res["wait_us_per_component"] = (st["host_wait_us"] - before["host_wait_us"]) / max(d, 1)
    r = {"layers": layers, "batch": batch, "logical_devices": devices, "policy": policy,
         "dynamic_ms": res["dynamic"], "dynamic_fused_ms": res["dynamic_fused"], "graph_ms": res["graph"],
         "dynamic_fused_dispatch_us_per_component": res["dynamic_fused_dispatch_us"],
         "dispatch_us_per_component": res["dispatch_us_per_component"],
         "wait_us_per_component": res["wait_us_per_component"]}
    rows.append(r)
    print(json.dumps(r), flush=True)
if len(sys.argv) > 1:
    json.dump(rows, open(sys.argv[1], "w"), indent=1)
