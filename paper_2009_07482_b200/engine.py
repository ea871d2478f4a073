"""The dispatch entry point as a Python object: a DAG template executed on one
B200 through the native engine (include/hetsim_c.h §3).

    eng = Engine(spec_text, params, batch=64, mode="graph")
    eng.bind(kernel, pos, host_array)                # per-instance input/output
    eng.bind(kernel, pos, weights, shared=True)      # resident weights (stride 0)
    ns = eng.run(first=0, n=4096)

Arrays may be numpy arrays or torch tensors (CPU, ideally pinned; or CUDA
tensors on the engine's GPU with on_device=True). The engine keeps a reference
to every bound array.
"""
from __future__ import annotations

import ctypes
import json

from ._native import HetsimError, check, lib


def _ptr_and_nbytes(arr):
    if hasattr(arr, "data_ptr"):  # torch
        return int(arr.data_ptr()), int(arr.numel() * arr.element_size()), bool(arr.is_cuda)
    if not arr.flags["C_CONTIGUOUS"]:
        raise ValueError("bound arrays must be C-contiguous")
    return int(arr.ctypes.data), int(arr.nbytes), False


class Engine:
    def __init__(self, spec_text: str, params: dict | None = None, *, gpu: int = 0, policy: str = "clustering",
                 mode: str = "graph", batch: int = 1, slots: int = 2, math: str = "tf32x3", cpu_devices=(),
                 fuse: int | bool = 3, trace: bool = False, device_gpus: dict | None = None,
                 domain_per_device: bool = False, dynamic_fuse: bool = False, deterministic: bool = False,
                 liveness: bool = True, ramp: int = 1, run_graph: bool = True, zero_copy: bool = True):
        """fuse (graph mode): 0 = one launch per ndrange; 1 = + grouped sibling GEMMs;
        2 = + chain rewrites (transpose -> gemm_nt, softmax as a GEMM epilogue, concat
        inputs written in place, fused attention heads); 3 (default, also True) = + each
        head's grouped Q/K/V projection absorbed into its attention launch (one
        HS_OP_HEAD launch per head component). Dynamic mode always launches per ndrange.
        trace: time every command of the first batch of each run with CUDA events
        (see trace(); graph mode issues that batch's plan directly instead of replaying it).
        device_gpus: {logical device id: GPU ordinal} places components on several GPUs
        (graph mode); an inter edge between GPUs becomes one peer copy over NVLink.
        domain_per_device: every logical device gets its own memory (test hook: the peer
        path on one GPU).
        dynamic_fuse: dynamic mode issues the graph plan's fused launches (per component)
        instead of one kernel per ndrange.
        deterministic: no atomic split-K anywhere (HS_FLAG_DETERMINISTIC). Single-instance
        GEMMs split K over a cluster and reduce in rank order either way; the flag only
        rules out the red.add fallback for tiles whose partial does not fit on chip.
        liveness: intermediate buffers share one arena per slot wherever the DAG orders
        all their accesses (False: one device allocation per output buffer).
        ramp (graph mode, host-memory bindings): the first and last chunks of a run are
        short so their copies are short: 1 = batch/4 instances, 0 = off, R > 1 = R.
        run_graph (graph mode, one GPU): a run that fits one batch replays a single graph
        holding its copies and the plan (one host submission per run).
        zero_copy (with run_graph, n == batch): per-instance inputs and outputs bound to
        dense memory on this GPU are read / written in place by the captured kernels
        (no copy-in / copy-out commands)."""
        fuse = 3 if fuse is True else int(fuse)
        cfg = {"spec": spec_text, "params": dict(params or {}), "gpu": gpu, "policy": policy, "mode": mode,
               "batch": batch, "slots": slots, "math": math, "cpu_devices": list(cpu_devices), "fuse": int(fuse),
               "trace": int(bool(trace)), "domain_per_device": int(bool(domain_per_device)),
               "dynamic_fuse": int(bool(dynamic_fuse)), "deterministic": int(bool(deterministic)),
               "liveness": int(bool(liveness)), "ramp": int(ramp), "run_graph": int(bool(run_graph)),
               "zero_copy": int(bool(zero_copy))}
        if device_gpus:
            cfg["device_gpus"] = {str(k): int(v) for k, v in device_gpus.items()}
        self._lib = lib()
        h = ctypes.c_void_p()
        check(self._lib.hs_engine_create(json.dumps(cfg).encode(), ctypes.byref(h)), "hs_engine_create")
        self._h = h
        self._keep = []
        self.batch = batch
        self.mode = mode

    def bind(self, kernel: int, pos: int, arr, *, shared: bool = False, stride_bytes: int | None = None):
        ptr, nbytes, on_dev = _ptr_and_nbytes(arr)
        if stride_bytes is None:
            if shared:
                stride_bytes = 0
            else:
                shape = tuple(arr.shape)
                stride_bytes = nbytes // shape[0] if shape and shape[0] else nbytes
        # instances the array holds: run() rejects [first, first+n) beyond it
        count = nbytes // stride_bytes if stride_bytes else 0
        check(self._lib.hs_engine_bind(self._h, kernel, pos, ctypes.c_void_p(ptr), stride_bytes, count, int(on_dev)),
              "hs_engine_bind")
        self._keep.append(arr)

    def run(self, first: int = 0, n: int = 1) -> int:
        ns = ctypes.c_int64(0)
        check(self._lib.hs_engine_run(self._h, first, n, ctypes.byref(ns)), "hs_engine_run")
        return ns.value

    def info(self, what: str = "plan") -> dict:
        p = ctypes.c_void_p()
        check(self._lib.hs_engine_info(self._h, what.encode(), ctypes.byref(p)), "hs_engine_info")
        try:
            return json.loads(ctypes.string_at(p).decode())
        finally:
            self._lib.hs_free_string(p)

    def trace(self) -> list[dict]:
        """SPEC.md:435 trace records of the last run's first batch: dicts with event, kind
        (write|ndrange|read), label (w1/e2/r1), kernel, component, device, queue, channel,
        start, finish (ms from the run's start event). Requires trace=True."""
        return self.info("trace")["trace"]

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            self._lib.hs_engine_destroy(self._h)
            self._h = ctypes.c_void_p()
        self._keep.clear()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def launch_count() -> int:
    """Node kernels launched through hs_launch in this process (graph replays not included)."""
    return int(lib().hs_launch_count())


__all__ = ["Engine", "HetsimError", "launch_count"]
