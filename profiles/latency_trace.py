"""Where the latency configs spend their time: the engine's per-command CUDA-event
trace (trace=True: the first batch's plan issued directly) of C1 / C2 / C3, device-
resident inputs, printed as (start, finish, duration) per command in us.
usage: python profiles/latency_trace.py [C1|C2|C3]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2009_07482_b200.engine import Engine  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C1"
text, params, arrays, outs, n, shared, io = bench.config_spec(cfg, 3, 9 if cfg == "C3" else 1)
dev = {k: torch.from_numpy(np.ascontiguousarray(a)).cuda() for k, a in arrays.items()}
out_dev = {(k, p): torch.zeros(n, e, device="cuda") for k, p, e in outs}
torch.cuda.synchronize()
with Engine(text, params, batch=n, slots=1, mode="graph", trace=True) as eng:
    for key, t in dev.items():
        eng.bind(*key, t, shared=key in shared or t.dim() == 1)
    for key, t in out_dev.items():
        eng.bind(*key, t)
    for _ in range(5):
        ns = eng.run(0, n)
    tr = eng.trace()
    print(f"{cfg}: traced run {ns / 1e3:.1f} us (direct issue with an event pair per command)")
    for r in sorted(tr, key=lambda r: r["start"]):
        d = (r["finish"] - r["start"]) * 1e3
        print(f"  {r['start'] * 1e3:8.2f} {r['finish'] * 1e3:8.2f} {d:7.2f}  c{r['component']} q{r['queue']} "
              f"{r['kind']:7s} {r['label']:5s} k{r['kernel']}")
