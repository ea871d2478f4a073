"""End-to-end DAG execution on the B200 through the engine C ABI, checked
against the CPU oracle executor on the same DAGs and inputs (C1, C2, C3 and a
2-layer encoder), in both execution modes:
  * dynamic — Alg. 1 with real host callbacks (fine-grained, 3 queues/device)
  * graph   — the scheduler's plan captured as a CUDA graph, batched instances
plus scheduling parity: the GPU run's completion order replayed through the
CPU scheduler (product and oracle) reproduces the dispatch sequence exactly.
"""
import json

import numpy as np
import pytest

from paper_2009_07482_b200 import hetsim, workloads
from paper_2009_07482_b200.engine import Engine

pytestmark = pytest.mark.gpu

TOL = 1e-4


def _normwise(y, ref):
    y, ref = np.asarray(y, np.float64), np.asarray(ref, np.float64)
    return float(np.max(np.abs(y - ref)) / max(np.max(np.abs(ref)), 1e-30))


def _encoder_arrays(meta, params, n):
    x = workloads.encoder_inputs(meta, params, n).reshape(n, -1)
    arrays = {(i["kernel"], i["pos"]): x for i in meta["x_inputs"]}
    for key, w in workloads.encoder_weights(meta).items():
        arrays[key] = w.reshape(-1)
    return arrays


def _run_gpu(text, params, arrays, n, **kw):
    outs = {(k, p): np.zeros((n, e), np.float32) for k, p, e in workloads.isolated_outputs(text, params)}
    with Engine(text, params, **kw) as eng:
        for key, arr in arrays.items():
            eng.bind(*key, arr, shared=arr.ndim == 1)
        for key, arr in outs.items():
            eng.bind(*key, arr)
        eng.run(0, n)
        info = eng.info("completions")
        plan = eng.info("plan")
    return outs, info, plan


CONFIGS = {
    "c1_fork_join": lambda: workloads.fork_join(),
    "c2_attention": lambda: workloads.attention(),
}


@pytest.mark.parametrize("name", sorted(CONFIGS))
@pytest.mark.parametrize("mode", ["dynamic", "graph"])
def test_small_configs(name, mode, oracle_mod):
    text, params = CONFIGS[name]()
    n = 3
    arrays = workloads.generic_inputs(text, params, n)
    ref = oracle_mod.run_dag(text, params, arrays, n)
    outs, _, _ = _run_gpu(text, params, arrays, n, mode=mode, batch=2)
    for key, r in ref.items():
        for i in range(n):
            assert _normwise(outs[key][i], r[i]) <= TOL, (key, i)


@pytest.mark.parametrize("mode,tc_mode,queues", [("graph", "per_head", 3), ("dynamic", "per_head", 3),
                                                 ("graph", "single", 1), ("graph", "per_kernel", 1)])
def test_encoder_layer(mode, tc_mode, queues, oracle_mod):
    text, params, meta = workloads.encoder(layers=1, tc_mode=tc_mode, queues=queues)
    n = 2
    arrays = _encoder_arrays(meta, params, n)
    ref = oracle_mod.run_dag(text, params, arrays, n)
    outs, _, plan = _run_gpu(text, params, arrays, n, mode=mode, batch=2)
    key = (meta["output"]["kernel"], meta["output"]["pos"])
    for i in range(n):
        assert _normwise(outs[key][i], ref[key][i]) <= TOL
    assert plan["kernels"] == 69


def test_two_layer_encoder_batched_graph(oracle_mod):
    text, params, meta = workloads.encoder(layers=2)
    n = 5  # two batches of 3 with a ragged tail, alternating slots
    arrays = _encoder_arrays(meta, params, n)
    ref = oracle_mod.run_dag(text, params, arrays, n)
    outs, _, _ = _run_gpu(text, params, arrays, n, mode="graph", batch=3, slots=2)
    key = (meta["output"]["kernel"], meta["output"]["pos"])
    for i in range(n):
        assert _normwise(outs[key][i], ref[key][i]) <= TOL


def test_grouped_sibling_gemms_match_unfused(oracle_mod):
    """Graph mode groups each head's Q/K/V projections (3 x N=64, shared X) into one
    N=192 tcgen05 launch; results equal the unfused launches and the oracle."""
    text, params, meta = workloads.encoder(layers=2)
    n = 3
    arrays = _encoder_arrays(meta, params, n)
    ref = oracle_mod.run_dag(text, params, arrays, n)
    key = (meta["output"]["kernel"], meta["output"]["pos"])
    fused, _, plan = _run_gpu(text, params, arrays, n, mode="graph", batch=3, fuse=1)
    plain, _, plan0 = _run_gpu(text, params, arrays, n, mode="graph", batch=3, fuse=0)
    assert plan["grouped_launches"] == 16 and plan0["grouped_launches"] == 0  # 8 heads x 2 layers
    assert plan["launches_per_batch"] == plan0["launches_per_batch"] - 32
    for i in range(n):
        assert _normwise(fused[key][i], ref[key][i]) <= TOL
        assert _normwise(fused[key][i], plain[key][i]) <= 1e-6


@pytest.mark.parametrize("math", ["tf32x3", "bf16x3"])
def test_chain_rewrites_match_oracle(math, oracle_mod):
    """fuse=2 (default): per head the transpose folds into a gemm_nt, the softmax
    becomes the QK^T GEMM's epilogue, the 8 Z_h GEMMs write the concat in place
    and each head's QK^T -> P·V -> C·W_h chain runs as one fused attn_head launch:
    33 launches fewer per layer, same results within tolerance."""
    text, params, meta = workloads.encoder(layers=2)
    n = 3
    arrays = _encoder_arrays(meta, params, n)
    ref = oracle_mod.run_dag(text, params, arrays, n)
    key = (meta["output"]["kernel"], meta["output"]["pos"])
    chained, _, plan = _run_gpu(text, params, arrays, n, mode="graph", batch=2, fuse=2, math=math)
    grouped, _, plan1 = _run_gpu(text, params, arrays, n, mode="graph", batch=2, fuse=1, math=math)
    assert plan["chain_rewrites"] == {"attention_head": 16, "concat_in_place": 2, "softmax_epilogue": 16,
                                      "transpose_into_gemm_nt": 16}
    assert plan1["chain_rewrites"] == {}
    assert plan["launches_per_batch"] == plan1["launches_per_batch"] - 66
    for i in range(n):
        assert _normwise(chained[key][i], ref[key][i]) <= TOL
        assert _normwise(chained[key][i], grouped[key][i]) <= 1e-5
    # fuse=3: each head's grouped Q/K/V launch is absorbed into a whole-head launch
    # (tf32 planes only); HS_OP_HEAD accumulates the P·V terms in another order, so it
    # agrees with the two launches it replaces to fp32 rounding
    whole, _, plan3 = _run_gpu(text, params, arrays, n, mode="graph", batch=2, fuse=3, math=math)
    heads = 16 if math == "tf32x3" else 0
    assert plan3["chain_rewrites"].get("head_fused", 0) == heads
    assert plan3["launches_per_batch"] == plan["launches_per_batch"] - heads
    for i in range(n):
        assert _normwise(whole[key][i], ref[key][i]) <= TOL
        assert _normwise(whole[key][i], chained[key][i]) <= 1e-5


@pytest.mark.parametrize("mode", ["graph", "dynamic"])
def test_encoder_bf16x3_within_tolerance(mode, oracle_mod):
    """BF16X3 math (resident-weight GEMMs as 3-term bf16 splits on kind::f16) stays
    within the 1e-4 fp32 tolerance on a 2-layer encoder (tests/split_precision_study.py
    predicts ~5e-6 for 12 layers)."""
    text, params, meta = workloads.encoder(layers=2)
    n = 2
    arrays = _encoder_arrays(meta, params, n)
    ref = oracle_mod.run_dag(text, params, arrays, n)
    key = (meta["output"]["kernel"], meta["output"]["pos"])
    outs, _, _ = _run_gpu(text, params, arrays, n, mode=mode, batch=2, math="bf16x3")
    for i in range(n):
        assert _normwise(outs[key][i], ref[key][i]) <= TOL


@pytest.mark.parametrize("policy,layers,devices", [("clustering", 1, 2), ("eager", 1, 2), ("heft", 1, 2),
                                                    ("clustering", 2, 3), ("eager", 2, 3), ("heft", 2, 3)])
def test_dynamic_completion_log_replays_identically(policy, layers, devices, oracle_mod):
    """Bit-exact scheduling parity for every policy: the completion order observed on
    the GPU, fed back through the CPU scheduler (product and oracle restatement),
    reproduces the GPU run's dispatch sequence (eager and HEFT see one component per
    kernel, so their logs are long and callback-driven)."""
    text, params, meta = workloads.encoder(layers=layers, devices=devices)
    arrays = _encoder_arrays(meta, params, 1)
    _, info, _ = _run_gpu(text, params, arrays, 1, mode="dynamic", batch=1, policy=policy)
    log = info["completions"]
    assert log and info["dispatches"]
    spec = hetsim.parse_spec(text, params)
    replay = hetsim.run_schedule(spec, policy=policy, replay=log)
    assert replay["dispatches"] == info["dispatches"]
    o = oracle_mod.schedule(oracle_mod.Spec(text, params), policy=policy, replay=log)
    assert o["dispatches"] == info["dispatches"]
    assert o["kernel_finish_order"] == replay["kernel_finish_order"]


@pytest.mark.parametrize("mode", ["graph", "dynamic"])
def test_spec_level_attn_head_nodes(mode, oracle_mod):
    """A DAG written with `attn_head` nodes (one per head: 4 kernels per head
    instead of 8) runs in both modes and matches the oracle."""
    text, params, meta = workloads.encoder(layers=2, fused_heads=True)
    n = 3
    arrays = _encoder_arrays(meta, params, n)
    ref = oracle_mod.run_dag(text, params, arrays, n)
    key = (meta["output"]["kernel"], meta["output"]["pos"])
    outs, _, plan = _run_gpu(text, params, arrays, n, mode=mode, batch=2)
    assert plan["kernels"] == 74
    for i in range(n):
        assert _normwise(outs[key][i], ref[key][i]) <= TOL


def test_trace_records_every_command_in_both_modes(oracle_mod):
    """trace=True: a CUDA-event pair around every command of the first batch.
    Same command count in both modes, queue order respected, outputs unchanged,
    and the device gaps between components are larger in dynamic mode (host
    callback round trip) than in graph mode (event join)."""
    from paper_2009_07482_b200 import reporting as R
    import statistics
    text, params, meta = workloads.encoder(layers=1)
    n = 2
    arrays = _encoder_arrays(meta, params, n)
    ref = oracle_mod.run_dag(text, params, arrays, n)
    key = (meta["output"]["kernel"], meta["output"]["pos"])
    med = {}
    counts = {}
    for mode in ("dynamic", "graph"):
        outs = {(k, p): np.zeros((n, e), np.float32) for k, p, e in workloads.isolated_outputs(text, params)}
        with Engine(text, params, mode=mode, batch=n, trace=True) as eng:
            for k, arr in arrays.items():
                eng.bind(*k, arr, shared=arr.ndim == 1)
            for k, arr in outs.items():
                eng.bind(*k, arr)
            eng.run(0, n)
            tr = eng.trace()
            disp = [c for c, _ in eng.info("trace")["dispatches"]]
        for i in range(n):
            assert _normwise(outs[key][i], ref[key][i]) <= TOL
        assert sum(r["kind"] == "ndrange" for r in tr) == 69
        assert all(0 <= r["start"] <= r["finish"] for r in tr)
        assert R.audit_queue_order(tr) == []
        counts[mode] = len(tr)
        med[mode] = statistics.median(g["gap"] for g in R.component_gaps(tr, disp))
    assert counts["dynamic"] == counts["graph"]
    assert med["dynamic"] > med["graph"], med


@pytest.mark.parametrize("fuse", [0, 3])
def test_components_across_memory_domains(fuse, oracle_mod):
    """components mapped to different GPUs. Every logical device gets its
    own memory domain (domain_per_device: the multi-GPU placement on this 1-GPU box),
    so each inter edge between components is one peer copy issued on the consumer's
    dependent write. Outputs equal the single-domain engine bit for bit (same
    kernels; a copy is exact) and match the oracle."""
    text, params, meta = workloads.encoder(layers=2, devices=9)
    n = 3
    arrays = _encoder_arrays(meta, params, n)
    ref = oracle_mod.run_dag(text, params, arrays, n)
    key = (meta["output"]["kernel"], meta["output"]["pos"])
    one, _, plan1 = _run_gpu(text, params, arrays, n, mode="graph", batch=2, fuse=fuse)
    many, _, plan = _run_gpu(text, params, arrays, n, mode="graph", batch=2, fuse=fuse,
                             device_gpus={d: 0 for d in range(9)}, domain_per_device=True)
    assert plan1["memory_domains"] == 1 and plan1["peer_copies_per_batch"] == 0
    assert plan["memory_domains"] == 9 and plan["peer_copies_per_batch"] > 0 and plan["captured"] == 1
    assert np.array_equal(many[key], one[key])
    for i in range(n):
        assert _normwise(many[key][i], ref[key][i]) <= TOL


def test_memory_domains_need_graph_mode():
    text, params, meta = workloads.encoder(layers=1, devices=2)
    with pytest.raises(Exception, match="graph mode"):
        Engine(text, params, mode="dynamic", device_gpus={0: 0, 1: 0}, domain_per_device=True)


@pytest.mark.parametrize("S,D,DFF", [(100, 256, 512), (64, 128, 256)])
def test_ragged_encoder_through_all_rewrites(S, D, DFF, oracle_mod):
    """Encoder shapes other than the C3 ones (S < 128 rows, narrower d_model / d_ff)
    through the default plan (whole-head kernels, concat in place, split-K for the
    single-instance batch) against the oracle, in one- and two-instance batches."""
    params = {"S": S, "D": D, "DK": 64, "DFF": DFF}
    text, params, meta = workloads.encoder(layers=2, heads=D // 64, params=params)
    key = (meta["output"]["kernel"], meta["output"]["pos"])
    for n, batch in ((1, 1), (3, 2)):
        arrays = _encoder_arrays(meta, params, n)
        ref = oracle_mod.run_dag(text, params, arrays, n)
        outs, _, plan = _run_gpu(text, params, arrays, n, mode="graph", batch=batch)
        assert plan["chain_rewrites"].get("head_fused", 0) == 2 * (D // 64)
        for i in range(n):
            assert _normwise(outs[key][i], ref[key][i]) <= TOL, (n, i)


def test_ramp_chunks_match_full_batches(oracle_mod):
    """Host-fed graph runs start and end with batch/4-instance chunks (a second
    captured graph) so the exposed copies are short; every instance is computed
    exactly as in the full-batch plan (bit-identical to the device-resident run,
    which has no ramp)."""
    import torch
    text, params, meta = workloads.encoder(layers=1)
    n, batch = 40, 8
    arrays = _encoder_arrays(meta, params, n)
    key = (meta["output"]["kernel"], meta["output"]["pos"])
    host, _, plan = _run_gpu(text, params, arrays, n, mode="graph", batch=batch, slots=3)
    assert plan["ramp_batch"] == 2
    x = torch.from_numpy(arrays[(meta["x_inputs"][0]["kernel"], meta["x_inputs"][0]["pos"])]).cuda()
    out = torch.zeros(n, params["S"] * params["D"], device="cuda")
    torch.cuda.synchronize()
    with Engine(text, params, mode="graph", batch=batch, slots=3) as eng:
        for i in meta["x_inputs"]:
            eng.bind(i["kernel"], i["pos"], x)
        for k, w in workloads.encoder_weights(meta).items():
            eng.bind(*k, w.reshape(-1), shared=True)
        eng.bind(*key, out)
        eng.run(0, n)
        assert eng.info("plan")["ramp_batch"] == 0
    assert np.array_equal(host[key], out.cpu().numpy())
    ref = oracle_mod.run_dag(text, params, {k: (v[:2] if v.ndim == 2 else v) for k, v in arrays.items()}, 2)
    for i in range(2):
        assert _normwise(host[key][i], ref[key][i]) <= TOL


def test_full_depth_c5_dag_matches_oracle(oracle_mod):
    """The C5 DAG at full depth (12 layers, 828 kernels) through the default plan,
    five instances in batches of two (a ragged last batch, three slots, ramp chunks
    off since n < 4 batches), every instance within 1e-4 of the CPU oracle."""
    text, params, meta = workloads.encoder(layers=12)
    n = 5
    arrays = _encoder_arrays(meta, params, n)
    ref = oracle_mod.run_dag(text, params, arrays, n)
    key = (meta["output"]["kernel"], meta["output"]["pos"])
    outs, _, plan = _run_gpu(text, params, arrays, n, mode="graph", batch=2, slots=3)
    assert plan["kernels"] == 828 and plan["launches_per_batch"] == 144
    for i in range(n):
        assert _normwise(outs[key][i], ref[key][i]) <= TOL, i


def test_production_stream_c5_sampled_parity(oracle_mod):
    """The bench's production configuration — 12 layers, batch 512, 3 slots — over
    2100 instances: device-resident (4 full batches and a ragged one rotating over
    the 3 slots) and host-fed through pinned memory (ramp chunks of 128 at both
    ends). Host-fed equals device-resident bit for bit on every instance; the first
    and last instance of every batch and ramp chunk, plus evenly spaced ones, are
    within 1e-4 of the fp32 CPU oracle and of the fp64 truth."""
    import torch
    text, params, meta = workloads.encoder(layers=12)
    n, batch = 2100, 512
    S, D = params["S"], params["D"]
    key = (meta["output"]["kernel"], meta["output"]["pos"])
    x = workloads.encoder_inputs(meta, params, n).reshape(n, -1)
    weights = workloads.encoder_weights(meta)

    def run(xb, out):
        with Engine(text, params, mode="graph", batch=batch, slots=3) as eng:
            for i in meta["x_inputs"]:
                eng.bind(i["kernel"], i["pos"], xb)
            for k, w in weights.items():
                eng.bind(*k, w.reshape(-1), shared=True)
            eng.bind(*key, out)
            eng.run(0, n)
            eng.run(0, n)  # a second pass through the same slots
            return eng.info("plan")

    x_dev = torch.from_numpy(x).cuda()
    out_dev = torch.zeros(n, S * D, device="cuda")
    torch.cuda.synchronize()
    plan = run(x_dev, out_dev)
    assert plan["ramp_batch"] == 0 and plan["launches_per_batch"] == 144
    dev = out_dev.cpu().numpy()
    del x_dev, out_dev
    torch.cuda.empty_cache()
    x_host = torch.from_numpy(x).pin_memory()
    out_host = torch.zeros(n, S * D).pin_memory()
    plan = run(x_host, out_host)
    assert plan["ramp_batch"] == 128
    assert np.array_equal(out_host.numpy(), dev)
    # batches of the device run: [0,512) .. [2048,2100); chunks of the host run:
    # [0,128), then 512-wide from 128, then 128-wide tail chunks from 1664
    edges = {0, 511, 512, 1023, 1024, 1535, 1536, 2047, 2048, 2099, 127, 128, 639, 640, 1663, 1664, 1791, 1792, 2047}
    idx = sorted(edges | set(np.linspace(0, n - 1, 8).round().astype(int).tolist()))
    xs = x[idx]
    arrays = {(i["kernel"], i["pos"]): xs for i in meta["x_inputs"]}
    for k, w in weights.items():
        arrays[k] = w.reshape(-1)
    ref = oracle_mod.run_dag(text, params, arrays, len(idx))[key]
    truth = oracle_mod.run_dag_f64(text, params, arrays, len(idx))[key]
    for j, i in enumerate(idx):
        assert _normwise(dev[i], ref[j]) <= TOL, i
        assert _normwise(dev[i], truth[j]) <= TOL, i


def test_single_term_tf32_plan(oracle_mod):
    """math='tf32' (one MMA per product, ~1e-3): the same plan (whole-head kernels,
    single-term pair GEMMs) runs and stays within its looser tolerance."""
    text, params, meta = workloads.encoder(layers=2)
    n = 3
    arrays = _encoder_arrays(meta, params, n)
    ref = oracle_mod.run_dag(text, params, arrays, n)
    key = (meta["output"]["kernel"], meta["output"]["pos"])
    outs, _, plan = _run_gpu(text, params, arrays, n, mode="graph", batch=2, math="tf32")
    assert plan["chain_rewrites"].get("head_fused") == 16
    for i in range(n):
        assert _normwise(outs[key][i], ref[key][i]) <= 5e-3


def test_peer_enable_same_gpu_is_a_noop():
    import ctypes
    from paper_2009_07482_b200 import _native
    L = _native.lib()
    a, b = ctypes.c_void_p(), ctypes.c_void_p()
    _native.check(L.hs_ctx_create(0, ctypes.byref(a)))
    _native.check(L.hs_ctx_create(0, ctypes.byref(b)))
    _native.check(L.hs_ctx_enable_peer(a, b))
    L.hs_ctx_destroy(a)
    L.hs_ctx_destroy(b)


@pytest.mark.parametrize("policy", ["clustering", "eager", "heft"])
def test_dynamic_mode_with_fused_launches(policy, oracle_mod):
    """dynamic_fuse: Alg. 1 with host callbacks, but each dispatched component issues
    the graph plan's fused launches (whole heads, grouped / chained GEMMs). Same
    kernels as graph mode, so the outputs are bit-identical to it."""
    text, params, meta = workloads.encoder(layers=2, devices=3)
    n = 3
    arrays = _encoder_arrays(meta, params, n)
    key = (meta["output"]["kernel"], meta["output"]["pos"])
    graph, _, _ = _run_gpu(text, params, arrays, n, mode="graph", batch=3)
    dyn, info, plan = _run_gpu(text, params, arrays, n, mode="dynamic", batch=3, policy=policy, dynamic_fuse=True)
    assert plan["dynamic_fused"] == 1 and plan["chain_rewrites"].get("head_fused") == 16
    assert np.array_equal(dyn[key], graph[key])
    ref = oracle_mod.run_dag(text, params, arrays, 1)
    assert _normwise(dyn[key][0], ref[key][0]) <= TOL
