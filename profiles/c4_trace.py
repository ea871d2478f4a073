"""C4 (6 layers x 64 instances) traced once: per-command CUDA-event times, the union of
kernel busy time vs the makespan, and the gaps on the critical chain of each layer."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2009_07482_b200 import reporting as R  # noqa: E402
from paper_2009_07482_b200.engine import Engine  # noqa: E402

text, params, arrays, outs, n, shared, io = bench.config_spec("C4", 3, 9)
out_arr = {(k, p): np.zeros((n, e), np.float32) for k, p, e in outs}
with Engine(text, params, batch=n, slots=1, mode="graph", trace=True) as eng:
    for key, a in arrays.items():
        eng.bind(*key, a, shared=key in shared)
    for key, a in out_arr.items():
        eng.bind(*key, a)
    eng.run(0, n)
    eng.run(0, n)
    tr = eng.trace()
nd = sorted([r for r in tr if r["kind"] == "ndrange" and r["finish"] - r["start"] > 0.0005], key=lambda r: r["start"])
busy, cur_s, cur_f = 0.0, None, None
for r in nd:
    if cur_f is None or r["start"] > cur_f:
        if cur_f is not None:
            busy += cur_f - cur_s
        cur_s, cur_f = r["start"], r["finish"]
    else:
        cur_f = max(cur_f, r["finish"])
busy += cur_f - cur_s
ms = R.makespan(tr)
print(json.dumps({"makespan_ms_traced": ms, "kernel_busy_union_ms": busy, "idle_ms": ms - busy,
                  "kernels": len(nd)}))
for r in nd[:40]:
    print(f"{r['start']:.4f} {r['finish']:.4f} {r['finish'] - r['start']:.4f} k{r['kernel']} c{r['component']} d{r['device']} q{r['queue']}")
