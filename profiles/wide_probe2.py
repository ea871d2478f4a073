"""Production-stream consistency probe: 12 layers, batch 512, 3 slots, device-resident
vs host-fed (ramp) outputs over n instances; rows that differ and their oracle error."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2009_07482_b200 import workloads  # noqa: E402
from paper_2009_07482_b200.engine import Engine  # noqa: E402
from oracle import oracle as O  # noqa: E402
layers = int(sys.argv[1]) if len(sys.argv) > 1 else 12
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2100
text, params, meta = workloads.encoder(layers=layers)
x = workloads.encoder_inputs(meta, params, n).reshape(n, -1)
key = (meta["output"]["kernel"], meta["output"]["pos"])
W = workloads.encoder_weights(meta)
def run(xb, out):
    with Engine(text, params, mode="graph", batch=512, slots=3) as eng:
        for i in meta["x_inputs"]: eng.bind(i["kernel"], i["pos"], xb)
        for k, w in W.items(): eng.bind(*k, w.reshape(-1), shared=True)
        eng.bind(*key, out)
        eng.run(0, n)
        eng.run(0, n)
xd = torch.from_numpy(x).cuda(); od = torch.zeros(n, 65536, device="cuda"); torch.cuda.synchronize()
run(xd, od); dev = od.cpu().numpy()
xh = torch.from_numpy(x).pin_memory(); oh = torch.zeros(n, 65536).pin_memory()
run(xh, oh); host = oh.numpy()
bad = np.where(~(dev == host).all(axis=1))[0]
print("rows differing:", len(bad), bad[:8], bad[-8:])
idx = sorted(set([int(i) for i in bad[:3]] + [int(i) for i in bad[-3:]] + [0, n - 1]))
arr = {(i["kernel"], i["pos"]): x[idx] for i in meta["x_inputs"]}
for k, w in W.items(): arr[k] = w.reshape(-1)
ref = O.run_dag(text, params, arr, len(idx))[key]
for j, i in enumerate(idx):
    e = lambda y: float(np.abs(y - ref[j]).max() / np.abs(ref[j]).max())
    print(i, "dev", e(dev[i]), "host", e(host[i]))
