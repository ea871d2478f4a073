"""End-to-end (pinned host buffers) C5 time per 4096-instance step against the ramp
chunk size, beside the device-resident time. usage: python profiles/e2e_ramp.py"""
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


def timed(xb, out, ramp, reps=3):
    with Engine(text, params, mode="graph", batch=B, slots=3, ramp=ramp) as eng:
        for i in meta["x_inputs"]:
            eng.bind(i["kernel"], i["pos"], xb)
        for k, w in W.items():
            eng.bind(*k, w.reshape(-1), shared=True)
        eng.bind(*key, out)
        eng.run(0, n)
        ts = [eng.run(0, n) / 1e6 for _ in range(reps)]
        return min(ts), eng.info("plan").get("ramp_batch")


xd = torch.from_numpy(x).cuda()
od = torch.empty(n, x.shape[1], device="cuda")
print(f"device-resident: {timed(xd, od, 1)[0]:.1f} ms")
xh = torch.from_numpy(x).pin_memory()
oh = torch.empty(n, x.shape[1]).pin_memory()
for r in (0, 1, 64, 256):
    ms, rb = timed(xh, oh, r)
    print(f"host-fed ramp={r} (ramp_batch {rb}): {ms:.1f} ms")
