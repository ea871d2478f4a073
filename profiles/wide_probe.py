import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2009_07482_b200 import workloads
from paper_2009_07482_b200.engine import Engine
from oracle import oracle as O
text, params, meta = workloads.encoder(layers=1)
n = 300
x = workloads.encoder_inputs(meta, params, n).reshape(n, -1)
key = (meta["output"]["kernel"], meta["output"]["pos"])
W = workloads.encoder_weights(meta)
def run(batch, slots=3):
    out = np.zeros((n, 65536), np.float32)
    with Engine(text, params, mode="graph", batch=batch, slots=slots) as eng:
        for i in meta["x_inputs"]: eng.bind(i["kernel"], i["pos"], x)
        for k, w in W.items(): eng.bind(*k, w.reshape(-1), shared=True)
        eng.bind(*key, out)
        eng.run(0, n)
    return out
a = run(128); b = run(64); c = run(300)
bad = np.where(~(a == c).all(axis=1))[0]
print("128 vs 300 rows differing:", len(bad), bad[:10], bad[-5:] if len(bad) else "")
bad2 = np.where(~(b == c).all(axis=1))[0]
print("64 vs 300 rows differing:", len(bad2), bad2[:10])
idx = [0, 127, 128, 255, 256, 299]
arr = {(i["kernel"], i["pos"]): x[idx] for i in meta["x_inputs"]}
for k, w in W.items(): arr[k] = w.reshape(-1)
ref = O.run_dag(text, params, arr, len(idx))[key]
for j, i in enumerate(idx):
    e = lambda y: float(np.abs(y - ref[j]).max() / np.abs(ref[j]).max())
    print(i, "err128", e(a[i]), "err300", e(c[i]), "err64", e(b[i]))
