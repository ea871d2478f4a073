"""Which bindings the whole-run graph uses in place (engine stats) for C1-C3."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2009_07482_b200.engine import Engine  # noqa: E402

for cfg, dev in (("C1", 1), ("C2", 1), ("C3", 9)):
    text, params, arrays, outs, n, shared, io = bench.config_spec(cfg, 3, dev)
    dt = {k: torch.from_numpy(np.ascontiguousarray(a)).cuda() for k, a in arrays.items()}
    od = {(k, p): torch.zeros(n, e, device="cuda") for k, p, e in outs}
    with Engine(text, params, batch=n, slots=1, mode="graph") as eng:
        for key, t in dt.items():
            eng.bind(*key, t, shared=key in shared or t.dim() == 1)
        for key, t in od.items():
            eng.bind(*key, t)
        eng.run(0, n)
        st = eng.info("stats")
    print(cfg, {k: st[k] for k in ("zero_copy_groups", "zero_copy_outputs")},
          "per-instance inputs:", sum(1 for k, t in dt.items() if not (k in shared or t.dim() == 1)), "outputs:", len(od))
