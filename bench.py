#!/usr/bin/env python
"""hetsim-b200 benchmark — BASELINE.json metric:
"DAG makespan (ms) and inference DAGs/sec at 1/2/4/8 B200 vs roofline & CPU".

Workload (config C5, BASELINE.json configs[4]): a 12-layer transformer-encoder
DAG (8 heads, d_model 512, seq 128, d_ff 2048; 828 kernels / 1103 edges / 108
task components, fine-grained: 3 command queues per device, clustering policy)
over a stream of 4096 independent instances, partitioned contiguously across
the ranks (one process per GPU, no collective on the data path). One step =
the whole 4096-instance stream; ms_per_step is its makespan (max over ranks)
and value = 4096 / makespan [DAGs/s].

  value  device-resident: X (1 GiB) and outputs live in HBM, copied per batch
         into the engine's slots (D2D) inside the timed region
  e2e    the same through the public engine API with pinned HOST buffers:
         H2D of every batch's X and D2H of every output inside the timed region

Usage: python bench.py [--gpus N --steps K --warmup W] [--impl reference]
Multi-GPU: `python bench.py --gpus N` re-launches itself as N ranks under
torch.distributed.run (the driver's own `torchrun ... bench.py --gpus N` works too).
Each rank checks >= 16 sampled instances of its own output against the CPU oracle.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import pathlib
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "DAG makespan (ms) and inference DAGs/sec at 1/2/4/8 B200 vs roofline & CPU"
UNIT = "DAGs/s"
TOTAL_INSTANCES = 4096
LAYERS = 12


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--instances", type=int, default=TOTAL_INSTANCES)
    ap.add_argument("--layers", type=int, default=LAYERS)
    ap.add_argument("--batch", type=int, default=0,
                    help="instances per batched node launch (0: min(512, half of this rank's instances), so every "
                         "rank pipelines at least two batches through its slots)")
    ap.add_argument("--slots", type=int, default=3, help="instance slots (graphs) in flight: copies of one batch overlap the others")
    ap.add_argument("--queues", type=int, default=3)
    ap.add_argument("--devices", type=int, default=1, help="logical devices in the cq map (all on this GPU)")
    ap.add_argument("--math", default="tf32x3")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-alt", action="store_true", help="skip the alternate-math measurement")
    ap.add_argument("--no-makespans", action="store_true", help="skip the C1-C4 makespan block")
    return ap.parse_args()


# --------------------------------------------------------------------------- helpers

def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu = gpu
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        rows = []
        try:
            for line in open(self.path):
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        except OSError:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        loaded = [s for s in sm if s > 0.5 * smax] or sm
        pw = [float(r[3]) for r in rows if r[3].replace(".", "").isdigit() and float(r[1] or 0) > 0.5 * smax]
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": smax, "reasons": reasons, "samples": len(rows),
                "power_w": statistics.median(pw) if pw else None}


def dist_setup():
    """One process per GPU (torchrun env). HS_BENCH_SHARED_GPU=1 is a test hook for
    1-GPU boxes: every rank drives cuda:0 and the timing collectives use gloo, so the
    multi-rank logic (partition, barrier, max over ranks) runs end to end."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        if os.environ.get("HS_BENCH_SHARED_GPU") == "1":
            local = 0
            torch.cuda.set_device(0)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def reduce_max(world, x, local):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cpu" if dist.get_backend() == "gloo" else f"cuda:{local}"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather(world, obj):
    """All ranks' `obj` (a small dict) on every rank."""
    if world == 1:
        return [obj]
    import torch.distributed as dist
    out = [None] * world
    dist.all_gather_object(out, obj)
    return out


def partition(total, world, rank):
    per = math.ceil(total / world)
    first = min(total, rank * per)
    return first, max(0, min(per, total - first))


# --------------------------------------------------------------------------- CPU arms (oracle port)

def cpu_sample(layers, n_inst=1, reps=1):
    """The CPU restatement (oracle/: clustering scheduler + fp32 kernels) on a bounded
    sample of the same workload; returns (instances/s, threads, seconds)."""
    from oracle import oracle as O
    from paper_2009_07482_b200 import workloads
    text, params, meta = workloads.encoder(layers=layers)
    x = workloads.encoder_inputs(meta, params, n_inst).reshape(n_inst, -1)
    arrays = {(i["kernel"], i["pos"]): x for i in meta["x_inputs"]}
    for k, w in workloads.encoder_weights(meta).items():
        arrays[k] = w.reshape(-1)
    spec = O.Spec(text, params)
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        O.schedule(spec)  # the restated Alg. 1 (clustering) decides the dispatch order
        O.run_dag(text, params, arrays, n_inst)
        times.append(time.perf_counter() - t0)
    t = min(times)
    return n_inst / t, O.max_threads(), t


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def cpu_threads():
    from oracle import oracle as O
    return O.max_threads()


def host_path_timing(layers, reps=5):
    """The host half of the path on the C5 template (828 kernels, 1103 edges): parse_spec +
    derive_components + classify_edges + bottom_level_ranks, timed single-threaded for
    the reference's own compiled L0-L2 (oracle/_ref) and for this repo's C++ runtime
    (hs_query), same JSON in, best of `reps`. The reference has no setup_cq /
    scheduler; ours adds the full Alg. 1 clustering plan (setup_cq per dispatch)."""
    from oracle import oracle as O
    from paper_2009_07482_b200 import _native, workloads
    text, params, _ = workloads.encoder(layers=layers)
    times = {}
    reqs = {"analyze": {"op": "analyze", "spec": text, "params": params},
            "ranks": {"op": "ranks", "spec": text, "params": params,
                      "times": {str(k): "1" for k in range(69 * layers)}}}
    for name, req in reqs.items():
        for who, fn in (("reference", O.ref_query if O.ref_available() else None), ("ours", _native.query)):
            if fn is None:
                continue
            best = 1e9
            for _ in range(reps):
                t0 = time.perf_counter()
                fn(req)
                best = min(best, time.perf_counter() - t0)
            times[f"{who}_{name}_ms"] = best * 1e3
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        _native.query({"op": "schedule", "spec": text, "params": params, "policy": "clustering"})
        best = min(best, time.perf_counter() - t0)
    times["ours_schedule_ms"] = best * 1e3
    times["note"] = ("single thread, JSON spec in; reference = /root/reference L0-L2 compiled unmodified "
                     "(oracle/_ref); 'schedule' = Alg. 1 clustering with setup_cq for every component")
    return times


def run_reference(args, world, rank):
    if rank != 0:
        return
    layers = args.layers
    vals = []
    # 12 instances per step: enough independent work to keep every host thread busy
    # (the same sample as the cpu_baseline of the GPU arm), ~1.5 s per step
    for i in range(args.warmup + args.steps):
        v, threads, t = cpu_sample(layers, n_inst=12)
        if i >= args.warmup:
            vals.append(v)
    v = statistics.mean(vals)
    sample = f"12 instances of the {layers}-layer encoder DAG per step (CPU oracle port: clustering + fp32 kernels)"
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 12 * 1000.0 / v,  # one step = the 12-instance sample
        "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"C5 {layers}-layer encoder DAG stream, {args.instances} instances (CPU sample)",
                   "instances": args.instances, "layers": layers, "kernels": 69 * layers},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample,
                         "cpu_model": cpu_model()},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- GPU arm

def nominal_tc(achieved, clocks, math):
    """The tensor pipe's issue-rate ceiling at the run's median SM clock: tcgen05
    kind::tf32 retires 4096 dense flop/clk/SM and kind::f16 8192 (profiles/mma_rate.cu
    measures both at full rate, M = 128, N = 64-256), / 3 MMAs per product. The
    measured-peak P above is lower (cuBLAS bf16 under the power cap)."""
    mhz = (clocks or {}).get("sm_mhz")
    if not mhz:
        return None
    per_clk = 8192 if math == "bf16x3" else 4096
    pk = per_clk * 148 * mhz * 1e6 / 1e12 / (1.0 if math == "tf32" else 3.0)
    return {"peak_at_sm_clock": pk, "sm_mhz": mhz, "flop_per_clk_per_sm": per_clk, "frac": achieved / pk}


def gemm_roofline(batch, math_mode, reps=20):
    """Time the dominant kernel exactly as the DAG launches it — FFN1, gemm_relu
    128x2048x512 per instance, batched, resident weight pre-split into planes —
    on its own stream with CUDA events around `reps` launches (after warm-up).
    Returns (achieved TFLOP/s, ms per launch, algorithmic FLOP per launch)."""
    import ctypes

    import torch

    from paper_2009_07482_b200 import _native
    L = _native.lib()
    code = {"tf32x3": 0, "tf32": 1, "simt": 2, "bf16x3": 3}[math_mode]
    M, N, K = 128, 2048, 512
    A = torch.randn(batch, M * K, device="cuda")
    W = torch.randn(K * N, device="cuda")
    C = torch.empty(batch, M * N, device="cuda")
    planes = torch.empty(2 * N * K, device="cuda")
    torch.cuda.synchronize()
    ctx, st, e0, e1 = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
    _native.check(L.hs_ctx_create(torch.cuda.current_device(), ctypes.byref(ctx)))
    _native.check(L.hs_stream_create(ctx, 0, ctypes.byref(st)))
    _native.check(L.hs_event_create(ctx, 1, ctypes.byref(e0)))
    _native.check(L.hs_event_create(ctx, 1, ctypes.byref(e1)))
    _native.check(L.hs_gemm_split_weights_ex(st, W.data_ptr(), 0, N, K, planes.data_ptr(), N * K,
                                             1 if math_mode == "bf16x3" else 0))
    a = _native.OpArgs()
    a.n_in = 2
    a.in_[0], a.in_[1] = A.data_ptr(), W.data_ptr()
    a.in_stride[0], a.in_stride[1] = M * K, 0
    a.out, a.out_stride = C.data_ptr(), M * N
    a.dims[0], a.dims[1], a.dims[2] = M, N, K
    a.aux = planes.data_ptr()
    for _ in range(3):
        _native.check(L.hs_launch(st, 2, ctypes.byref(a), code, batch))
    _native.check(L.hs_stream_sync(st))
    _native.check(L.hs_event_record(e0, st))
    for _ in range(reps):
        _native.check(L.hs_launch(st, 2, ctypes.byref(a), code, batch))
    _native.check(L.hs_event_record(e1, st))
    _native.check(L.hs_event_sync(e1))
    ns = ctypes.c_int64()
    _native.check(L.hs_event_elapsed_ns(e0, e1, ctypes.byref(ns)))
    t = ns.value / 1e9 / reps
    flops = 2.0 * M * N * K * batch
    for h in (e0, e1):
        L.hs_event_destroy(h)
    L.hs_stream_destroy(st)
    L.hs_ctx_destroy(ctx)
    return flops / t / 1e12, t * 1e3, flops


def _time_launches(L, st, launch, reps):
    """CUDA events on the launching stream around `reps` launches (after 3 warm-up)."""
    import ctypes

    from paper_2009_07482_b200 import _native
    ctx, e0, e1 = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
    _native.check(L.hs_ctx_create(0, ctypes.byref(ctx)))
    _native.check(L.hs_event_create(ctx, 1, ctypes.byref(e0)))
    _native.check(L.hs_event_create(ctx, 1, ctypes.byref(e1)))
    for _ in range(3):
        launch()
    _native.check(L.hs_stream_sync(st))
    _native.check(L.hs_event_record(e0, st))
    for _ in range(reps):
        launch()
    _native.check(L.hs_event_record(e1, st))
    _native.check(L.hs_event_sync(e1))
    ns = ctypes.c_int64()
    _native.check(L.hs_event_elapsed_ns(e0, e1, ctypes.byref(ns)))
    for h in (e0, e1):
        L.hs_event_destroy(h)
    L.hs_ctx_destroy(ctx)
    return ns.value / 1e9 / reps


def _traffic(name, batch, math_mode="tf32x3"):
    """DRAM bytes per launch from a committed ncu --set full capture (profiles/<name>),
    scaled to `batch` instances; None when absent."""
    f = ROOT / "profiles" / name
    if not f.exists():
        return None
    per = json.loads(f.read_text()).get(math_mode, {}).get("dram_bytes_per_launch_per_instance")
    return per * batch if per else None


def kernel_rooflines(batch, peak_tflops, hbm_gbs, reps=20):
    """The other two kernels of the C5 plan, launched as the DAG launches them:
    the whole-head kernel (HS_OP_HEAD, tensor-bound; algorithmic flops of the head
    chain, 2*S*192*D + 2*2*S*S*64 + 2*S*64*64 per instance) and add_layernorm
    (HBM-bound; 3*R*C*4 + 8*C bytes per instance)."""
    import ctypes

    import torch

    from paper_2009_07482_b200 import _native
    L = _native.lib()
    S, D, dk = 128, 512, 64
    ctx, st = ctypes.c_void_p(), ctypes.c_void_p()
    _native.check(L.hs_ctx_create(0, ctypes.byref(ctx)))
    _native.check(L.hs_stream_create(ctx, 0, ctypes.byref(st)))
    X = torch.randn(batch, S * D, device="cuda")
    Wqkv = torch.randn(3, D * dk, device="cuda") / 22.6
    Wh = torch.randn(dk * dk, device="cuda") / 8
    pq = torch.empty(2 * 3 * dk * D, device="cuda")
    Z = torch.empty(batch, S * dk, device="cuda")
    torch.cuda.synchronize()
    for m in range(3):
        _native.check(L.hs_gemm_split_weights_strided(st, Wqkv[m].data_ptr(), 0, dk, D, pq.data_ptr() + 4 * m * dk * D,
                                                      3 * dk * D))
    ph = torch.empty(2 * dk * dk, device="cuda")
    torch.cuda.synchronize()
    _native.check(L.hs_gemm_split_weights(st, Wh.data_ptr(), 0, dk, dk, ph.data_ptr()))
    h = _native.OpArgs()
    h.n_in = 2
    h.in_[0], h.in_stride[0] = X.data_ptr(), S * D
    h.in_[1], h.in_stride[1] = ph.data_ptr(), 0
    h.aux = pq.data_ptr()
    h.out, h.out_stride = Z.data_ptr(), S * dk
    h.dims[0], h.dims[1], h.dims[2] = S, D, dk
    h.fparam[0] = 0.125
    t_head = _time_launches(L, st, lambda: _native.check(L.hs_launch(st, 10, ctypes.byref(h), 0, batch)), reps)
    f_head = batch * (2.0 * S * 3 * dk * D + 2.0 * 2 * S * S * dk + 2.0 * S * dk * dk)
    A, B2, Y = (torch.randn(batch, S * D, device="cuda") for _ in range(3))
    g, be = torch.ones(D, device="cuda"), torch.zeros(D, device="cuda")
    torch.cuda.synchronize()
    a = _native.OpArgs()
    a.n_in = 4
    for i, t in enumerate((A, B2, g, be)):
        a.in_[i], a.in_stride[i] = t.data_ptr(), (0 if t.dim() == 1 else S * D)
    a.out, a.out_stride = Y.data_ptr(), S * D
    a.dims[0], a.dims[1] = S, D
    a.fparam[0], a.fparam[1] = 1.0, 1e-5
    t_ln = _time_launches(L, st, lambda: _native.check(L.hs_launch(st, 7, ctypes.byref(a), 0, batch)), reps)
    b_ln = batch * (3.0 * S * D * 4) + 8.0 * D
    L.hs_stream_destroy(st)
    L.hs_ctx_destroy(ctx)
    return [
        {"kernel": f"head_kernel (HS_OP_HEAD: Q/K/V projection + attention, 2 instances in flight per SM) x{batch}",
         "bound": "tensor", "achieved": f_head / t_head / 1e12, "peak": peak_tflops, "unit": "TFLOP/s",
         "frac": f_head / t_head / 1e12 / peak_tflops, "ms_per_launch": t_head * 1e3,
         "traffic": _traffic("head_traffic.json", batch),
         "note": "algorithmic flops of the head chain"},
        {"kernel": f"add_ln_kernel x{batch}", "bound": "hbm", "achieved": b_ln / t_ln / 1e9, "peak": hbm_gbs,
         "unit": "GB/s", "frac": b_ln / t_ln / 1e9 / hbm_gbs, "ms_per_launch": t_ln * 1e3},
    ]


def matmul_peak(dtype):
    """cuBLAS dense throughput at 8192^3 in-run: torch.float32 with TF32 enabled, or bf16."""
    import torch
    torch.backends.cuda.matmul.allow_tf32 = True
    n = 8192
    a = torch.randn(n, n, device="cuda", dtype=dtype)
    b = torch.randn(n, n, device="cuda", dtype=dtype)
    for _ in range(3):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch.matmul(a, b)
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    torch.backends.cuda.matmul.allow_tf32 = False
    del a, b
    return 2.0 * n ** 3 / best / 1e12


def sample_instances(n, batch, ramp, count=16):
    """Rank-local instances whose outputs are checked against the CPU oracle: the first
    and last instance of every batch (even and odd positions, i.e. both CTAs of a pair),
    the last instance of the first ramp chunk and the first of the next chunk (host-fed
    runs), topped up with evenly spaced instances to at least `count`."""
    import numpy as np
    s = set()
    for b in range(math.ceil(n / batch)):
        s.update((b * batch, min(n, (b + 1) * batch) - 1))
    if ramp:
        s.update((min(n - 1, ramp - 1), min(n - 1, ramp)))
    for i in np.linspace(0, n - 1, count).round().astype(int):
        if len(s) >= count:
            break
        s.add(int(i))
    return sorted(s)


def oracle_rows(layers, instances):
    """CPU oracle outputs for the given global instance indices: (fp32 oracle [k, S*D]
    (sequential-k GEMMs), fp64 truth [k, S*D])."""
    import numpy as np

    from oracle import oracle as O
    from paper_2009_07482_b200 import workloads
    text, params, meta = workloads.encoder(layers=layers)
    x = np.concatenate([workloads.encoder_inputs(meta, params, 1, first=i).reshape(1, -1) for i in instances])
    arrays = {(i["kernel"], i["pos"]): x for i in meta["x_inputs"]}
    for k, w in workloads.encoder_weights(meta).items():
        arrays[k] = w.reshape(-1)
    key = (meta["output"]["kernel"], meta["output"]["pos"])
    return O.run_dag(text, params, arrays, len(instances))[key], O.run_dag_f64(text, params, arrays, len(instances))[key]


def errors(y, ref32, ref64):
    """Per-row errors, maxed over rows: normwise |y-ref|_inf/|ref|_inf against the fp32
    oracle and the fp64 truth, elementwise |y-ref|/max(|ref|, 1e-6), and the fp32
    oracle's own normwise distance from the truth (the headroom reference)."""
    import numpy as np
    y, r32, r64 = (np.asarray(a, np.float64).reshape(len(a), -1) for a in (y, ref32, ref64))

    def nw(a, b):
        return float((np.abs(a - b).max(axis=1) / np.maximum(np.abs(b).max(axis=1), 1e-30)).max())
    return {"normwise_vs_oracle": nw(y, r32), "normwise_vs_f64": nw(y, r64),
            "elementwise_vs_oracle": float((np.abs(y - r32) / np.maximum(np.abs(r32), 1e-6)).max()),
            "oracle_normwise_vs_f64": nw(r32, r64)}


def config_spec(cfg, queues=3, devices=1):
    """(spec_text, params, per-instance inputs {key: [n, e] or shared [e]}, output keys, n_instances, shared keys,
    io bytes per instance) for BASELINE.json configs C1-C4 (workloads.py)."""
    from paper_2009_07482_b200 import workloads
    if cfg in ("C1", "C2"):
        text, params = workloads.fork_join(queues=queues) if cfg == "C1" else workloads.attention(queues=queues)
        arrays = workloads.generic_inputs(text, params, 1)
        outs = [(k, p, e) for k, p, e in workloads.isolated_outputs(text, params)]
        io = 4 * (sum(a.shape[1] for a in arrays.values()) + sum(e for _, _, e in outs))
        return text, params, arrays, outs, 1, [], io
    layers, n = (1, 1) if cfg == "C3" else (6, 64)
    text, params, meta = workloads.encoder(layers=layers, queues=queues, devices=devices)
    x = workloads.encoder_inputs(meta, params, n).reshape(n, -1)
    arrays = {(i["kernel"], i["pos"]): x for i in meta["x_inputs"]}
    shared = []
    for key, w in workloads.encoder_weights(meta).items():
        arrays[key] = w.reshape(-1)
        shared.append(key)
    outs = [(meta["output"]["kernel"], meta["output"]["pos"], params["S"] * params["D"])]
    return text, params, arrays, outs, n, shared, 2 * x.shape[1] * 4


def config_makespan(cfg, fuse=3, queues=3, devices=1, reps=20, warmup=3, math_mode="tf32x3", check=True, batch=None,
                    slots=1, host_io=False, **engine_kw):
    """Makespan of one whole run of config `cfg` (all its instances in one batch) in graph
    mode with device-resident inputs/outputs: median over `reps` runs of the engine's own
    CUDA-event timing (start event -> end event on the origin stream, which joins every
    queue stream). Returns the makespan, T* (roofline.dag_bound) and T*/makespan; with
    `check`, instance 0's outputs are compared with the CPU oracle (normwise, 1e-4)."""
    import numpy as np
    import torch

    from paper_2009_07482_b200 import roofline
    from paper_2009_07482_b200.engine import Engine
    text, params, arrays, outs, n, shared, io = config_spec(cfg, queues, devices)
    # host_io: inputs and outputs in pinned host memory (every run copies them in and out,
    # the paper's isolated writes / reads over PCIe); otherwise device-resident, which a
    # one-batch run reads and writes in place (engine zero_copy)
    place = (lambda t: t.pin_memory()) if host_io else (lambda t: t.cuda())
    dev = {}
    x_cache = {}
    for key, a in arrays.items():
        if id(a) not in x_cache:
            x_cache[id(a)] = place(torch.from_numpy(np.ascontiguousarray(a)))
        dev[key] = x_cache[id(a)]
    out_dev = {(k, p): place(torch.zeros(n, e)) for k, p, e in outs}
    torch.cuda.synchronize()
    batch = batch or n
    with Engine(text, params, batch=batch, slots=slots, mode="graph", fuse=fuse, math=math_mode, **engine_kw) as eng:
        for key, t in dev.items():
            eng.bind(*key, t, shared=key in shared or t.dim() == 1)
        for key, t in out_dev.items():
            eng.bind(*key, t)
        for _ in range(warmup):
            eng.run(0, n)
        ns = [eng.run(0, n) for _ in range(reps)]
        launches = eng.info("plan").get("launches_per_batch")
    ms = statistics.median(ns) / 1e6
    pk, _ = peaks()
    P = pk["bf16_tflops"] / 2.0 / 3.0 if math_mode != "bf16x3" else pk["bf16_tflops"] / 3.0
    bound = roofline.dag_bound(text, params, n, P, pk["hbm_gbs"], shared_inputs=shared, io_bytes=io)
    r = {"config": cfg, "instances": n, "batch": batch, "slots": slots, "fuse": fuse, "queues": queues, "logical_devices": devices, "math": math_mode,
         "launches": launches, "makespan_ms": ms, "makespan_min_ms": min(ns) / 1e6, "t_star_ms": bound["t_star_ms"],
         "bound": bound["bound"], "frac": bound["t_star_ms"] / ms}
    if check:  # every instance of the config against the fp32 oracle and the fp64 truth
        from oracle import oracle as O
        t0 = time.perf_counter()
        ref = O.run_dag(text, params, arrays, n)
        first_s = time.perf_counter() - t0
        # the CPU port's makespan for this config: best of the warm runs (three when a run is
        # short, where OpenMP wake-ups dominate; one for C4)
        runs = []
        for _ in range(3 if first_s < 0.5 else 1):
            t0 = time.perf_counter()
            O.run_dag(text, params, arrays, n)
            runs.append(time.perf_counter() - t0)
        r["cpu_port_ms"] = min(runs) * 1e3
        truth = O.run_dag_f64(text, params, arrays, n)
        errs = [errors(out_dev[k].cpu().numpy(), ref[k], truth[k]) for k in out_dev]
        r["parity"] = {key: max(e[key] for e in errs) for key in errs[0]}
        r["parity"]["instances_checked"] = n
        r["normwise_err_vs_cpu_oracle"] = r["parity"]["normwise_vs_oracle"]
    return r


def config_makespans():
    """BASELINE.json configs C1-C4 on this GPU: makespan of one run (all instances, one
    batch, graph mode, device-resident), T* and T*/makespan, parity of instance 0 vs the
    CPU oracle; plus the paper's fine- vs coarse-grained comparison:
    3 queues per device vs 1, with one launch per ndrange (fuse 0, the paper's execution)
    and with all launch rewrites (fuse 3)."""
    out = {}
    best = {"C1": {}, "C2": {}, "C3": {"devices": 9}, "C4": {"devices": 9}}
    for cfg, kw in best.items():
        r = config_makespan(cfg, **kw)
        out[cfg] = {k: r[k] for k in ("instances", "logical_devices", "queues", "fuse", "launches", "makespan_ms",
                                      "t_star_ms", "bound", "frac", "normwise_err_vs_cpu_oracle", "parity",
                                      "cpu_port_ms")}
        out[cfg]["gpu_speedup_vs_cpu_port"] = r["cpu_port_ms"] / r["makespan_ms"]
        rh = config_makespan(cfg, check=False, host_io=True, **kw)
        out[cfg]["makespan_host_io_ms"] = rh["makespan_ms"]
    out["C4"]["target_1p5x_t_star_ms"] = 1.5 * out["C4"]["t_star_ms"]
    grain = []
    for cfg in ("C3", "C4"):
        for fuse in (0, 3):
            for queues in (1, 3):
                r = config_makespan(cfg, fuse=fuse, queues=queues, devices=1, reps=10, check=False)
                grain.append({"config": cfg, "fuse": fuse, "queues": queues, "makespan_ms": r["makespan_ms"]})
    out["fine_vs_coarse"] = {"logical_devices": 1, "rows": grain,
                             "note": "queues=1 is the coarse-grained default mc=(1,0,0); queues=3 fine-grained"}
    out["note"] = ("median of 20 runs of the engine's CUDA-event makespan (start -> end event on the origin stream) "
                   "with device-resident inputs and outputs (a one-batch run replays one graph and uses them in place); "
                   "makespan_host_io_ms = the same with pinned host inputs / outputs copied in and out every run; "
                   "C3/C4 use one logical device per component of a layer (9) so that heads run concurrently; "
                   "cpu_port_ms = the same config (all instances) through the CPU oracle port (fp32 C kernels, "
                   f"{cpu_threads()} threads, {cpu_model()})")
    return out


def normwise(y, ref):
    import numpy as np
    y, ref = np.asarray(y, np.float64), np.asarray(ref, np.float64)
    return float(np.max(np.abs(y - ref)) / max(float(np.max(np.abs(ref))), 1e-30))


def run_ours(args, world, rank, local):
    import numpy as np
    import torch

    from paper_2009_07482_b200 import workloads
    from paper_2009_07482_b200.engine import Engine

    torch.cuda.set_device(local)
    text, params, meta = workloads.encoder(layers=args.layers, queues=args.queues, devices=args.devices)
    first, n = partition(args.instances, world, rank)
    if args.batch <= 0:  # same on every rank: derived from the largest partition
        per = math.ceil(args.instances / world)
        args.batch = max(1, min(512, math.ceil(per / 2)))
    S, D = params["S"], params["D"]
    inst_bytes = S * D * 4
    weights = workloads.encoder_weights(meta)
    x_np = workloads.encoder_inputs(meta, params, n, first=first).reshape(n, S * D)
    out_key = (meta["output"]["kernel"], meta["output"]["pos"])

    def make_engine(x, out, math_mode):
        eng = Engine(text, params, gpu=local, batch=args.batch, slots=args.slots, math=math_mode, mode="graph")
        for i in meta["x_inputs"]:
            eng.bind(i["kernel"], i["pos"], x)
        for key, w in weights.items():
            eng.bind(*key, w.reshape(-1), shared=True)
        eng.bind(*out_key, out)
        return eng

    def timed(eng, steps):
        tot = 0
        for _ in range(steps):
            tot += eng.run(0, n)
        return tot / 1e9

    def device_resident(math_mode, sample_clocks):
        """Device-resident arm: X and outputs in HBM. Returns (ms/step max over ranks, plan, stats,
        the rank's outputs copied to the host, clocks, all finite)."""
        x_dev = torch.from_numpy(x_np).cuda()
        out_dev = torch.empty(n, S * D, device="cuda")
        torch.cuda.synchronize()  # the engine's streams do not order after torch's
        eng = make_engine(x_dev, out_dev, math_mode)
        for _ in range(args.warmup):
            eng.run(0, n)
        barrier(world)
        torch.cuda.synchronize()
        clk = None
        if sample_clocks:
            with ClockSampler(local) as c:
                s = timed(eng, args.steps)
            clk = c.summary()
        else:
            s = timed(eng, args.steps)
        torch.cuda.synchronize()
        barrier(world)
        s = reduce_max(world, s, local)
        plan, stats = eng.info("plan"), eng.info("stats")
        out_np = out_dev.cpu().numpy()
        finite = bool(np.isfinite(out_np).all())
        eng.close()
        del x_dev, out_dev
        torch.cuda.empty_cache()
        return s / args.steps * 1e3, plan, stats, out_np, clk, finite

    ms_per_step, plan, stats, out_main, clocks, finite = device_resident(args.math, True)
    assert finite, "non-finite outputs"
    value = args.instances / (ms_per_step / 1e3)
    launches = int(stats["launches_per_batch"]) * math.ceil(n / args.batch) * args.steps

    # end-to-end arm through the public API with pinned host buffers
    e2e = None
    e2e_out = None
    ramp = 0
    if not args.no_e2e:
        x_host = torch.from_numpy(x_np).pin_memory()
        out_host = torch.empty(n, S * D).pin_memory()
        eng_h = make_engine(x_host, out_host, args.math)
        for _ in range(args.warmup):
            eng_h.run(0, n)
        barrier(world)
        torch.cuda.synchronize()
        e2e_s = timed(eng_h, args.steps)
        barrier(world)
        e2e_s = reduce_max(world, e2e_s, local)
        ramp = int(eng_h.info("plan").get("ramp_batch", 0))
        e2e = {"value": args.instances / (e2e_s / args.steps), "unit": UNIT,
               "h2d_bytes_per_step": args.instances * inst_bytes, "d2h_bytes_per_step": args.instances * inst_bytes,
               "ms_per_step": e2e_s / args.steps * 1e3, "ramp_batch": ramp}
        e2e_out = out_host.numpy()
        eng_h.close()
    alt = None
    if not args.no_alt:
        alt_math = "bf16x3" if args.math != "bf16x3" else "tf32x3"
        alt_ms, _, _, alt_out, alt_clk, alt_finite = device_resident(alt_math, True)
        alt = {"math": alt_math, "value": args.instances / (alt_ms / 1e3), "ms_per_step": alt_ms, "clocks": alt_clk,
               "finite": alt_finite}

    # Parity of this very run on every rank: sampled instances of the device-resident
    # output (every batch's first and last instance, ramp-chunk instances, >= 16) against
    # the fp32 CPU oracle and the fp64 truth; the host-fed e2e output must equal the
    # device-resident one bit for bit on every instance, and its sampled rows are checked too.
    t0 = time.perf_counter()
    idx = sample_instances(n, args.batch, ramp) if n else []
    par = {"rank": rank, "instances": [first + i for i in idx]}
    if idx:
        ref32, ref64 = oracle_rows(args.layers, par["instances"])
        par.update(errors(out_main[idx], ref32, ref64))
        if alt is not None:
            ae = errors(alt_out[idx], ref32, ref64)
            par["alt_normwise_vs_oracle"] = ae["normwise_vs_oracle"]
            par["alt_normwise_vs_f64"] = ae["normwise_vs_f64"]
        if e2e_out is not None:
            par["e2e_bit_identical_all_instances"] = bool(np.array_equal(e2e_out, out_main))
            par["e2e_normwise_vs_oracle"] = errors(e2e_out[idx], ref32, ref64)["normwise_vs_oracle"]
    par["oracle_s"] = time.perf_counter() - t0
    pars = gather(world, par)
    del out_main, e2e_out

    line = None
    if rank == 0:
        pk, pk_kind = peaks()
        tf32 = matmul_peak(torch.float32)
        achieved, ms_launch, flops = gemm_roofline(args.batch, args.math)
        if args.math == "bf16x3":
            bf16 = pk["bf16_tflops"]
            peak, peak_note = bf16 / 3.0, (f"MEASURED_PEAKS.json ({pk_kind}) dense bf16 burst {bf16:.0f} TFLOP/s "
                                           f"/ 3 MMAs per product")
        else:
            # tcgen05 kind::tf32 issues at half the kind::f16 rate: the dense TF32 peak is the
            # measured bf16 peak / 2 (cuBLAS's own TF32 GEMM, measured in-run, reaches less)
            tf32_peak = max(pk["bf16_tflops"] / 2.0, tf32)
            peak, peak_note = tf32_peak / 3.0, (
                f"TF32 dense peak = MEASURED_PEAKS.json ({pk_kind}) bf16 {pk['bf16_tflops']:.0f} / 2 = "
                f"{pk['bf16_tflops'] / 2:.0f} TFLOP/s (cuBLAS TF32 measured in-run: {tf32:.0f}); / 3 MMAs per product")
        # the same denominator from the sustained (4 s back-to-back, power-capped) bf16 figure
        bf16_sus = pk.get("bf16_tflops_sustained", pk["bf16_tflops"])
        peak_sus = bf16_sus / 3.0 if args.math == "bf16x3" else bf16_sus / 2.0 / 3.0
        traffic = None
        tf = ROOT / "profiles" / "ffn1_traffic.json"
        if tf.exists():
            t = json.loads(tf.read_text())
            traffic = t.get(args.math, {}).get("dram_bytes_per_launch_per_instance")
            traffic = traffic * args.batch if traffic else None
        checked = [p for p in pars if p["instances"]]
        worst = {k: max(p[k] for p in checked) for k in ("normwise_vs_oracle", "normwise_vs_f64",
                                                         "elementwise_vs_oracle", "oracle_normwise_vs_f64")}
        parity = {"math": args.math, "tol_normwise": 1e-4, "ranks": world,
                  "instances_checked": sum(len(p["instances"]) for p in checked), **worst,
                  "pass": worst["normwise_vs_oracle"] <= 1e-4,
                  "per_rank": pars,
                  "note": "max over the sampled instances of every rank; elementwise uses an absolute floor of 1e-6 "
                          "(near-zero LayerNorm outputs dominate it); oracle_normwise_vs_f64 = the fp32 oracle's own "
                          "distance from the float64 truth"}
        if not args.no_e2e:
            parity["e2e_bit_identical_all_instances"] = all(p.get("e2e_bit_identical_all_instances") for p in checked)
            parity["e2e_normwise_vs_oracle"] = max(p["e2e_normwise_vs_oracle"] for p in checked)
        if alt is not None:
            alt["normwise_err_vs_cpu_oracle"] = max(p["alt_normwise_vs_oracle"] for p in checked)
            alt["normwise_err_vs_f64"] = max(p["alt_normwise_vs_f64"] for p in checked)
            alt["instances_checked"] = sum(len(p["instances"]) for p in checked)
        cpu = None
        if not args.no_cpu_baseline:
            v, threads, t = cpu_sample(args.layers, n_inst=64)
            cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "port", "cpu_model": cpu_model(),
                   "sample": f"64 instances of the {args.layers}-layer DAG ({t:.1f} s; oracle port: clustering "
                             f"scheduler + fp32 kernels on all host threads)",
                   "host_path": host_path_timing(args.layers)}
        makespans = None if args.no_makespans else config_makespans()
        others = kernel_rooflines(args.batch, peak, pk["hbm_gbs"]) if args.math in ("tf32x3", "tf32") else None
        flop_per_inst = 782.2e6 * args.layers
        dtypes = {"tf32x3": "f32 (3xTF32 split on tcgen05, fp32-accurate)",
                  "bf16x3": "f32 (bf16x3 split on tcgen05 for weight GEMMs, 3xTF32 elsewhere; <=1e-4)",
                  "tf32": "tf32", "simt": "f32"}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": dtypes.get(args.math, args.math),
            "data": "synthetic (splitmix64 uniform inputs, random-init weights)",
            "config": {"workload": f"C5: {args.layers}-layer encoder DAG (8 heads, d_model 512, seq 128, d_ff 2048), "
                                   f"stream of {args.instances} instances",
                       "kernels_per_dag": plan["kernels"], "edges": plan["edges"], "components": plan["components"],
                       "policy": "clustering", "queues_per_device": args.queues, "logical_devices": args.devices,
                       "batch": args.batch, "slots": args.slots, "mode": "graph",
                       "grouped_launches_per_batch": plan.get("grouped_launches"),
                       "chain_rewrites_per_batch": plan.get("chain_rewrites"),
                       "launches_per_batch": plan.get("launches_per_batch"),
                       "parallelism": f"instance partition x{world}", "math": args.math,
                       "l2": "inputs (1 GiB X + 1 GiB out per step) larger than L2"},
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": f"gemm_pair_kernel (CTA pair, cta_group::2, 192-wide tiles, two TMEM accumulators) "
                                   f"FFN1 gemm_relu 128x2048x512 x{args.batch}, resident pre-split weight, {args.math} "
                                   f"({ms_launch:.3f} ms/launch)",
                         "peak_note": peak_note, "measured_peaks_file": pk_kind,
                         "nominal": nominal_tc(achieved, clocks, args.math)},
            "dag_roofline": {"flop_per_dag": flop_per_inst, "achieved_tflops": flop_per_inst * value / 1e12,
                             "frac_of_peak": flop_per_inst * value / 1e12 / (peak * world),
                             "t_star_ms": args.instances * flop_per_inst / (peak * world * 1e12) * 1e3,
                             "peak_sustained": peak_sus,
                             "t_star_sustained_ms": args.instances * flop_per_inst / (peak_sus * world * 1e12) * 1e3,
                             "frac_of_sustained_peak": flop_per_inst * value / 1e12 / (peak_sus * world),
                             "note": "T* = instances x flop/DAG / P (compute-bound, SURVEY.md 8d); frac_of_peak = T*/ms_per_step "
                                     "with P from the burst bf16 peak; the step is a long run under sw_power_cap, for which "
                                     "MEASURED_PEAKS.json's sustained bf16 figure is the matching denominator "
                                     "(peak_sustained, t_star_sustained_ms, frac_of_sustained_peak)"},
            "roofline_other_kernels": others,
            "makespans": makespans,
            "parity": parity,
            "alt_math": alt,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks,
            # the step runs under sw_power_cap: throughput per watt of board power
            "energy": ({"power_w": clocks["power_w"], "dags_per_joule": value / (clocks["power_w"] * world),
                        "note": "rank 0's median nvidia-smi power.draw over the timed region (a moving "
                                "average); DAGs per joule per GPU"}
                       if clocks and clocks.get("power_w") else None),
            "device_bytes": plan["device_bytes"],
        }
    return line


def spawn_ranks(n):
    """`bench.py --gpus N` outside torchrun: re-launch this command as N ranks (one per
    GPU, rank i on cuda:i) under torch.distributed.run on 127.0.0.1; rank 0 prints the line."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(pathlib.Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


def main():
    args = parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        sys.exit(spawn_ranks(args.gpus))
    world, rank, local = dist_setup()
    if args.impl == "ours" and world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; timing {world} rank(s)", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    line = run_ours(args, world, rank, local)
    if rank == 0 and line is not None:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        barrier(world)  # rank 0's baselines run after the timed regions
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
