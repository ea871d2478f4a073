"""Cross-process determinism of single-instance runs: hash of the C1 / C3 engine outputs
(graph mode, default options) and of a 256^3 single-instance GEMM; run this script twice
and compare the printed digests. usage: python profiles/determinism_probe.py"""
import hashlib
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2009_07482_b200.engine import Engine  # noqa: E402
from tests.gpu_util import launch  # noqa: E402
from tests.test_gpu_kernels import _rand, _t  # noqa: E402

for cfg, dev in (("C1", 1), ("C2", 1), ("C3", 9)):
    text, params, arrays, outs, n, shared, io = bench.config_spec(cfg, 3, dev)
    dt = {k: torch.from_numpy(np.ascontiguousarray(a)).cuda() for k, a in arrays.items()}
    od = {(k, p): torch.zeros(n, e, device="cuda") for k, p, e in outs}
    digs = []
    for det in (False, True):
        with Engine(text, params, batch=n, slots=1, mode="graph", deterministic=det) as eng:
            for key, t in dt.items():
                eng.bind(*key, t, shared=key in shared or t.dim() == 1)
            for key, t in od.items():
                eng.bind(*key, t)
            hs = set()
            for _ in range(5):
                eng.run(0, n)
                hs.add(hashlib.sha1(b"".join(t.cpu().numpy().tobytes() for t in od.values())).hexdigest()[:12])
        digs.append(sorted(hs))
    print(cfg, "default:", digs[0], "deterministic:", digs[1])
M = N = K = 256
A, B = _t(_rand(41, (1, M * K))), _t(_rand(42, (1, N * K)))
hs = set()
for _ in range(5):
    out = torch.full((1, M * N), float("nan"), device="cuda")
    launch("gemm", [A, B], out, [M, N, K], batch=1)
    hs.add(hashlib.sha1(out.cpu().numpy().tobytes()).hexdigest()[:12])
print("gemm 256^3:", sorted(hs))
