"""Per-step times of the C5 stream (4096 instances, batch 512, 3 slots): device-resident vs
host-fed (pinned) engines, alternated, 8 steps each after 3 warm-up steps. Shows whether the
end-to-end gap is systematic or a few slow steps. usage: python profiles/e2e_steps.py"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2009_07482_b200 import workloads  # noqa: E402
from paper_2009_07482_b200.engine import Engine  # noqa: E402

n, B = 4096, 512
text, params, meta = workloads.encoder(layers=12)
x = workloads.encoder_inputs(meta, params, 64).reshape(64, -1)
x = np.tile(x, (n // 64, 1))
W = workloads.encoder_weights(meta)
key = (meta["output"]["kernel"], meta["output"]["pos"])


def steps(xb, out, k=8):
    with Engine(text, params, mode="graph", batch=B, slots=3) as eng:
        for i in meta["x_inputs"]:
            eng.bind(i["kernel"], i["pos"], xb)
        for kk, w in W.items():
            eng.bind(*kk, w.reshape(-1), shared=True)
        eng.bind(*key, out)
        for _ in range(3):
            eng.run(0, n)
        return [eng.run(0, n) / 1e6 for _ in range(k)]


xd = torch.from_numpy(x).cuda()
od = torch.empty(n, x.shape[1], device="cuda")
xh = torch.from_numpy(x).pin_memory()
oh = torch.empty(n, x.shape[1]).pin_memory()
for rep in range(2):
    for name, xb, out in (("device", xd, od), ("host-fed", xh, oh)):
        t = steps(xb, out)
        print(f"{name:9s} mean {np.mean(t):7.2f} ms  min {min(t):7.2f}  max {max(t):7.2f}  steps " +
              " ".join(f"{v:.1f}" for v in t), flush=True)
