"""dynamic Alg. 1 policies (clustering / eager / HEFT) on the
B200 with measured host-callback cost, against graph mode (the same plan with
event joins instead of host round trips).

For each configuration: wall time of one run (CUDA events around the run),
makespan of the traced batch, and the device gaps between consecutive
components on a logical device (reporting.component_gaps): in dynamic mode a
gap is completion on the GPU -> cudaLaunchHostFunc -> MPSC queue ->
Scheduler::cb -> select -> setup_cq -> dispatch -> first kernel start.
usage: python profiles/callback_gaps.py [out.json]"""
import json
import statistics
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2009_07482_b200 import reporting as R, workloads  # noqa: E402
from paper_2009_07482_b200.engine import Engine  # noqa: E402


def run(layers, mode, policy, batch, devices, tc_mode="per_head"):
    text, params, meta = workloads.encoder(layers=layers, devices=devices, tc_mode=tc_mode)
    x = workloads.encoder_inputs(meta, params, batch).reshape(batch, -1)
    outs = {(k, p): np.zeros((batch, e), np.float32) for k, p, e in workloads.isolated_outputs(text, params)}
    with Engine(text, params, mode=mode, policy=policy, batch=batch, trace=True) as eng:
        for i in meta["x_inputs"]:
            eng.bind(i["kernel"], i["pos"], x)
        for k, w in workloads.encoder_weights(meta).items():
            eng.bind(*k, w.reshape(-1), shared=True)
        for k, arr in outs.items():
            eng.bind(*k, arr)
        eng.run(0, batch)  # warm-up (plan, capture, uploads)
        ns = eng.run(0, batch)
        info = eng.info("trace")
    tr, disp = info["trace"], [c for c, _ in info["dispatches"]]
    gaps = [g["gap"] for g in R.component_gaps(tr, disp)]
    return {"layers": layers, "mode": mode, "policy": policy, "batch": batch, "logical_devices": devices,
            "tc_mode": tc_mode, "run_ms": ns / 1e6, "traced_makespan_ms": R.makespan(tr),
            "components": len(disp), "gap_median_us": 1e3 * statistics.median(gaps) if gaps else None,
            "gap_mean_us": 1e3 * statistics.mean(gaps) if gaps else None,
            "gap_p90_us": 1e3 * float(np.percentile(gaps, 90)) if gaps else None}


rows = []
for layers, batch in ((1, 1), (6, 64)):
    for devices in (1, 2):
        for mode, policy in (("graph", "clustering"), ("dynamic", "clustering"), ("dynamic", "eager"),
                             ("dynamic", "heft")):
            r = run(layers, mode, policy, batch, devices)
            rows.append(r)
            print(json.dumps(r), flush=True)
# coarse vs fine grained (PAPER.md:341-355 analogue): one component per kernel, eager
for mode in ("graph", "dynamic"):
    r = run(1, mode, "eager", 1, 2, tc_mode="per_kernel")
    rows.append(r)
    print(json.dumps(r), flush=True)
if len(sys.argv) > 1:
    json.dump(rows, open(sys.argv[1], "w"), indent=1)
