"""platform_sim: the product's C++ simulator (hs_query
"simulate") against SPEC's worked examples and against the restatement in
oracle/platform_sim.py (exact rational equality of every trace record)."""
import json
import random
from fractions import Fraction

import pytest

from oracle import platform_sim as OS
from paper_2009_07482_b200 import _native, workloads
from tests.dag_gen import layered_dag


def sim(text, params, profiles, policy="clustering", cpu_devices=(), delay=0):
    req = {"op": "simulate", "spec": text, "params": params, "policy": policy, "cpu_devices": list(cpu_devices),
           "device_profiles": profiles, "callback_delay": str(delay)}
    return _native.query(req)["simulate"]


def by_label(trace):
    return {(r["component"], r["label"]): r for r in trace}


def kernel(kid, ins, outs, name="op", dev="gpu"):
    return {"id": kid, "name": name, "dev": dev, "workDimension": 1, "globalWorkSize": ["1", "1", "1"],
            "inputBuffers": [{"type": "float32", "size": s, "pos": p} for p, s in ins],
            "outputBuffers": [{"type": "float32", "size": s, "pos": p} for p, s in outs],
            "ioBuffers": [], "varArguments": []}


def doc(kernels, tc, queues, edges=(), devices=1):
    return json.dumps({"kernels": kernels, "tc": tc, "cq": [{"device": d, "queues": queues} for d in range(devices)],
                       "depends": [list(e) for e in edges]})


def gpu(times, channels=2, bw="1000", lat="0", shares=None, device=0):
    return {"device": device, "type": "gpu", "kernel_times": {str(k): str(v) for k, v in times.items()},
            "kernel_share": {str(k): str(v) for k, v in (shares or {}).items()}, "copy_channels": channels,
            "bandwidth": bw, "transfer_latency": lat}


# ------------------------------------------------------------------ SPEC.md worked examples

def test_transfer_time_examples():
    p = {"type": "gpu", "bandwidth": "10000", "transfer_latency": "1/10"}
    assert OS.transfer_time(1 << 20, p) == Fraction(1, 10) + Fraction(1 << 20, 10000)  # 0.1 + 104.8576 ms
    assert OS.transfer_time(12345, {"type": "cpu"}) == 0
    assert OS.transfer_time(0, p) == Fraction(1, 10)
    # product: one kernel with a 1 MiB isolated input (and a 4-byte isolated output)
    text = doc([kernel(0, [(0, str(1 << 18))], [(1, "1")])], [[0]], 1)
    r = sim(text, {}, [gpu({0: 3}, bw="10000", lat="1/10")])
    w = by_label(r["trace"])[(0, "w1")]
    assert Fraction(w["finish"]) - Fraction(w["start"]) == Fraction(1, 10) + Fraction(1 << 20, 10000)


def test_queue_order_and_cross_queue_dependency():
    # [w1, e1, r1] on one queue: e1 starts when w1 finishes (transfer 2 ms)
    text = doc([kernel(0, [(0, "500")], [(1, "500")])], [[0]], 1)
    r = by_label(sim(text, {}, [gpu({0: 5}, bw="1000")])["trace"])
    assert Fraction(r[(0, "w1")]["finish"]) == 2 and Fraction(r[(0, "e1")]["start"]) == 2
    assert Fraction(r[(0, "r1")]["start"]) == 7
    # k0 -> k1 intra edge on different queues: k1's ndrange waits for k0's (E_Q pair)
    text = doc([kernel(0, [], [(0, "1")]), kernel(1, [(0, "1")], [(1, "1")])], [[0, 1]], 2, edges=[(0, 0, 1, 0)])
    r = by_label(sim(text, {}, [gpu({0: 4, 1: 1}, bw="1000000")])["trace"])
    assert Fraction(r[(0, "e2")]["start"]) == Fraction(r[(0, "e1")]["finish"])


def test_two_writes_two_channels_start_together():
    text = doc([kernel(0, [(0, "250")], [(1, "1")]), kernel(1, [(0, "250")], [(1, "1")])], [[0, 1]], 2)
    r = by_label(sim(text, {}, [gpu({0: 1, 1: 1}, channels=2)])["trace"])
    w1, w2 = r[(0, "w1")], r[(0, "w2")]
    assert w1["start"] == w2["start"] == "0" and {w1["channel"], w2["channel"]} == {0, 1}


def test_channel_fifo_examples():
    # 1 channel, two 2 ms transfers: the second starts at 2
    text = doc([kernel(0, [(0, "500")], [(1, "1")]), kernel(1, [(0, "500")], [(1, "1")])], [[0, 1]], 2)
    r = by_label(sim(text, {}, [gpu({0: 1, 1: 1}, channels=1)])["trace"])
    assert sorted(Fraction(r[(0, w)]["start"]) for w in ("w1", "w2")) == [0, 2]
    # 3 transfers of 5, 5, 2 ms on 2 channels: the third starts at 5 on channel 0
    ks = [kernel(i, [(0, s)], [(1, "1")]) for i, s in enumerate(["1250", "1250", "500"])]
    r = by_label(sim(doc(ks, [[0, 1, 2]], 3), {}, [gpu({0: 1, 1: 1, 2: 1}, channels=2)])["trace"])
    w3 = r[(0, "w3")]
    assert Fraction(w3["start"]) == 5 and w3["channel"] == 0


@pytest.mark.parametrize("n,share,expect", [(1, "1/2", 10), (2, "1/2", 10), (3, "1/2", 15)])
def test_processor_sharing_examples(n, share, expect):
    # n independent 10 ms kernels with share s, co-started (CPU device: transfers are free)
    ks = [kernel(i, [], [(0, "1")], dev="cpu") for i in range(n)]
    text = doc(ks, [list(range(n))], n)
    prof = [{"device": 0, "type": "cpu", "kernel_times": {str(i): "10" for i in range(n)},
             "kernel_share": {str(i): share for i in range(n)}}]
    r = sim(text, {}, prof, cpu_devices=[0])
    nd = [e for e in r["trace"] if e["kind"] == "ndrange"]
    assert all(Fraction(e["start"]) == 0 and Fraction(e["finish"]) == expect for e in nd)


def test_single_queue_single_channel_is_serial_and_deterministic():
    text, params = workloads.fork_join(queues=1)
    prof = [gpu({0: 3, 1: 2, 2: 1, 3: 1}, channels=1, bw="100000")]
    a = sim(text, params, prof)
    b = sim(text, params, prof)
    assert a == b
    tr = sorted(a["trace"], key=lambda e: Fraction(e["start"]))
    for x, y in zip(tr, tr[1:]):
        assert Fraction(y["start"]) >= Fraction(x["finish"])


def test_errors():
    text, params = workloads.fork_join()
    with pytest.raises(_native.HetsimError) as e:
        sim(text, params, [gpu({0: 1, 1: 1, 2: 1})])  # kernel 3 has no time
    assert e.value.errc == "MissingProfileEntry"
    with pytest.raises(_native.HetsimError) as e:
        sim(text, params, [gpu({0: 1, 1: 1, 2: 1, 3: 1}, shares={0: 2})])
    assert e.value.errc == "InvalidParam"


# ------------------------------------------------------------------ product == restatement

def _oracle(text, params, profiles, policy, cpu_devices=(), delay=0):
    return OS.simulate(text, params, profiles, policy=policy, cpu_devices=cpu_devices, callback_delay=delay)


def _same(prod, orc):
    assert Fraction(prod["makespan"]) == orc["makespan"]
    assert [list(x) for x in prod["dispatches"]] == orc["schedule"]["dispatches"]
    assert len(prod["trace"]) == len(orc["trace"])
    for p, o in zip(prod["trace"], orc["trace"]):
        assert (p["component"], p["label"], p["kernel"], p["device"], p["queue"], p["channel"]) == \
            (o["component"], o["label"], o["kernel"], o["device"], o["queue"], o["channel"])
        assert Fraction(p["start"]) == o["start"] and Fraction(p["finish"]) == o["finish"]


def _random_profiles(rng, spec_text, devices, cpu_devices):
    kids = [k["id"] for k in json.loads(spec_text)["kernels"]]
    profs = []
    for d in range(devices):
        typ = "cpu" if d in cpu_devices else "gpu"
        profs.append({"device": d, "type": typ,
                      "kernel_times": {str(k): f"{rng.randint(1, 40)}/{rng.choice([1, 2, 4])}" for k in kids},
                      "kernel_share": {str(k): rng.choice(["1", "1/2", "1/4", "3/10"]) for k in kids},
                      "copy_channels": rng.randint(1, 3), "bandwidth": str(rng.choice([100, 1000, 4096])),
                      "transfer_latency": rng.choice(["0", "1/10", "1"])})
    # the scheduler reads per-type times from the first device of each type
    return profs


@pytest.mark.parametrize("seed", range(60))
def test_product_matches_restatement_random(seed):
    rng = random.Random(1000 + seed)
    cpu = seed % 3 == 0
    text, params = layered_dag(seed, max_kernels=14, devices=2, cpu_frac=0.4 if cpu else 0.0)
    cpu_devices = [1] if cpu else []
    profs = _random_profiles(rng, text, 2, cpu_devices)
    if cpu:  # same type -> same times on every device of that type
        pass
    policy = ["clustering", "eager", "heft"][seed % 3]
    delay = rng.choice(["0", "1/2", "3"])
    try:
        orc = _oracle(text, params, profs, policy, cpu_devices, Fraction(delay))
    except Exception as e:  # the product must fail the same way
        with pytest.raises(_native.HetsimError) as pe:
            sim(text, params, profs, policy, cpu_devices, delay)
        assert pe.value.errc == getattr(e, "errc", type(e).__name__)
        return
    _same(sim(text, params, profs, policy, cpu_devices, delay), orc)


def _fork_join_mapping(mask):
    """Fig. 1 fork-join with kernel i on the CPU when bit i of mask is set; one
    component per kernel, device 0 = GPU, device 1 = CPU (the 16 mappings of §1)."""
    text, params = workloads.fork_join(queues=2)
    d = json.loads(text)
    for k in d["kernels"]:
        k["dev"] = "cpu" if mask >> k["id"] & 1 else "gpu"
    d["tc"] = [[k["id"]] for k in d["kernels"]]
    d["cq"] = [{"device": 0, "queues": 2}, {"device": 1, "queues": 2}]
    return json.dumps(d), params


@pytest.mark.parametrize("profile", ["unit", "gpu_fast", "copy_bound"])
def test_fork_join_all_16_mappings(profile):
    """SPEC.md:560 acceptance 1: every mapping of Fig. 1's DAG, three profiles,
    product makespan == restatement makespan exactly."""
    gt = {"unit": (1, 1), "gpu_fast": (1, 20), "copy_bound": (4, 6)}[profile]
    for mask in range(16):
        text, params = _fork_join_mapping(mask)
        profs = [
            {"device": 0, "type": "gpu", "kernel_times": {str(k): str(gt[0]) for k in range(4)},
             "kernel_share": {"1": "1/2", "2": "1/2"}, "copy_channels": 2,
             "bandwidth": "65536" if profile != "copy_bound" else "8192", "transfer_latency": "1/10"},
            {"device": 1, "type": "cpu", "kernel_times": {str(k): str(gt[1]) for k in range(4)}},
        ]
        orc = _oracle(text, params, profs, "clustering", [1])
        _same(sim(text, params, profs, "clustering", [1]), orc)
