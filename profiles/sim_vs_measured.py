"""platform_sim on the CPU fed with kernel times measured on
the B200, against the makespans measured on the B200.

1. Standalone kernel times: a 2-layer encoder (batch 64) run with one queue,
   one launch per ndrange (fuse=0), every command timed with CUDA events.
2. Measured makespans of the traced batch: graph mode (3 queues, fuse=0) and
   dynamic mode (3 queues; host callbacks); the dynamic run also gives the
   median device gap between components (callback round trip).
3. Simulated makespans: the same DAG/partition through Alg. 1 + platform_sim
   (hs_query "simulate") with those kernel times (share 1: a B200 kernel fills
   the GPU), measured H2D bandwidth / latency, and callback_delay = 0 (graph)
   or the measured gap (dynamic). Dynamic mode is simulated twice: without and
   with the host dispatch cost (dispatch_cost = the engine's measured host time
   per component dispatch: stream/event setup and launches on the host thread).
usage: python profiles/sim_vs_measured.py [out.json]"""
import ctypes
import json
import statistics
import sys
import time
from fractions import Fraction

import numpy as np

sys.path.insert(0, ".")
from paper_2009_07482_b200 import _native, reporting as R, workloads  # noqa: E402
from paper_2009_07482_b200.engine import Engine  # noqa: E402

LAYERS, BATCH = 2, 64


def traced(queues, mode, fuse):
    text, params, meta = workloads.encoder(layers=LAYERS, queues=queues)
    x = workloads.encoder_inputs(meta, params, BATCH).reshape(BATCH, -1)
    outs = {(k, p): np.zeros((BATCH, e), np.float32) for k, p, e in workloads.isolated_outputs(text, params)}
    with Engine(text, params, mode=mode, batch=BATCH, trace=True, fuse=fuse) as eng:
        for i in meta["x_inputs"]:
            eng.bind(i["kernel"], i["pos"], x)
        for k, w in workloads.encoder_weights(meta).items():
            eng.bind(*k, w.reshape(-1), shared=True)
        for k, arr in outs.items():
            eng.bind(*k, arr)
        eng.run(0, BATCH)
        before = eng.info("stats")
        eng.run(0, BATCH)
        after = eng.info("stats")
        info = eng.info("trace")
    n = after["host_dispatches"] - before["host_dispatches"]
    cost = (after["host_dispatch_us"] - before["host_dispatch_us"]) / n / 1e3 if n else 0.0  # ms per dispatch
    return text, params, info["trace"], [c for c, _ in info["dispatches"]], cost


def h2d_profile():
    L = _native.lib()
    ctx, st = ctypes.c_void_p(), ctypes.c_void_p()
    _native.check(L.hs_ctx_create(0, ctypes.byref(ctx)))
    _native.check(L.hs_stream_create(ctx, 0, ctypes.byref(st)))
    res = {}
    for nbytes in (4096, 64 << 20):
        host, dev = ctypes.c_void_p(), ctypes.c_void_p()
        _native.check(L.hs_host_alloc(nbytes, ctypes.byref(host)))
        _native.check(L.hs_malloc(ctx, nbytes, ctypes.byref(dev)))
        for _ in range(3):
            _native.check(L.hs_memcpy_h2d(st, dev, host, nbytes))
        _native.check(L.hs_stream_sync(st))
        t0 = time.perf_counter()
        reps = 20
        for _ in range(reps):
            _native.check(L.hs_memcpy_h2d(st, dev, host, nbytes))
        _native.check(L.hs_stream_sync(st))
        res[nbytes] = (time.perf_counter() - t0) / reps * 1e3  # ms
        L.hs_free(ctx, dev)
        L.hs_host_free(host)
    lat = res[4096]
    bw = (64 << 20) / max(res[64 << 20] - lat, 1e-6)  # bytes / ms
    return lat, bw


def frac(ms):
    return str(Fraction(round(ms * 1e3), 1000))  # microsecond resolution keeps the rationals small


def main(out=None):
    _, _, solo, _, _ = traced(1, "graph", 0)
    ktime = {}
    for r in solo:
        if r["kind"] == "ndrange":
            ktime[r["kernel"]] = r["finish"] - r["start"]
    lat, bw = h2d_profile()
    rows = []
    for mode in ("graph", "dynamic"):
        text, params, tr, disp, cost = traced(3, mode, 0)
        gaps = [g["gap"] for g in R.component_gaps(tr, disp)]
        delay = statistics.median(gaps) if mode == "dynamic" else 0.0
        prof = [{"device": 0, "type": "gpu", "kernel_times": {str(k): frac(v) for k, v in ktime.items()},
                 "copy_channels": 2, "bandwidth": str(int(round(bw))), "transfer_latency": frac(lat)}]
        for with_cost in ((False, True) if mode == "dynamic" else (False,)):
            dc = cost if with_cost else 0.0
            s = _native.query({"op": "simulate", "spec": text, "params": params, "policy": "clustering",
                               "device_profiles": prof, "callback_delay": frac(delay),
                               "dispatch_cost": frac(dc)})["simulate"]
            meas = R.makespan(tr)
            row = {"mode": mode, "layers": LAYERS, "batch": BATCH, "queues": 3, "kernels": len(ktime),
                   "measured_makespan_ms": meas, "simulated_makespan_ms": s["makespan_ms"],
                   "sim_over_measured": s["makespan_ms"] / meas, "callback_delay_ms": delay,
                   "dispatch_cost_ms": dc, "h2d_latency_ms": lat, "h2d_GBps": bw / 1e6,
                   "sum_standalone_ms": sum(ktime.values())}
            rows.append(row)
            print(json.dumps(row), flush=True)
    if out:
        json.dump(rows, open(out, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else None)
