"""Paper Expt. 1 on the B200: clustering over mc = <q_gpu, q_cpu, h_cpu>
for transformer-head DAGs of H heads (beta = 256).

  simulated: sweep.sweep_clustering with node times measured here (B200 engine trace for
             the GPU, the oracle's C kernels for the host CPU) over the whole grid
  measured:  all heads on the B200, one launch per ndrange (the paper's execution model),
             q_gpu = 1..5 on one logical device, and with one logical device per head
usage: python profiles/expt1_sweep.py [out.json]"""
import json
import sys

sys.path.insert(0, ".")
from paper_2009_07482_b200 import sweep  # noqa: E402

BETA = 256
gpu_t, share = sweep.gpu_node_times(BETA)
cpu_t = sweep.cpu_node_times(BETA)
print(json.dumps({"gpu_node_ms": gpu_t, "gpu_share": share, "cpu_node_ms": cpu_t}), flush=True)
out = {"beta": BETA, "gpu_node_ms": gpu_t, "gpu_share": share, "cpu_node_ms": cpu_t, "simulated": [], "measured": []}
for H in (1, 2, 4, 8, 10):
    t = sweep.sweep_clustering(H, BETA, gpu_t, cpu_t, share, q_gpu=range(1, 6), q_cpu=range(1, 6))
    row = {"heads": H, "configs": len(t["rows"]), "default_ms": t["default"]["makespan_ms"],
           "best": t["best"]["mc"], "best_ms": t["best"]["makespan_ms"], "best_vs_default": t["best_vs_default"]}
    out["simulated"].append(row)
    print(json.dumps({"simulated": row}), flush=True)
    meas = {}
    for devices in (1, H):
        for q in range(1, 6):
            meas[f"d{devices}q{q}"] = sweep.measured_gpu_makespan(H, BETA, q, devices=devices)
    default = meas["d1q1"]
    best = min(meas, key=meas.get)
    mrow = {"heads": H, "makespans_ms": meas, "default_ms": default, "best": best, "best_ms": meas[best],
            "best_vs_default": default / meas[best]}
    out["measured"].append(mrow)
    print(json.dumps({"measured": mrow}), flush=True)
if len(sys.argv) > 1:
    json.dump(out, open(sys.argv[1], "w"), indent=1)
