"""Alg. 1 scheduler (no reference implementation exists).
Product C++ scheduler vs the independent Python restatement (oracle/oracle.py)
on random DAGs for all three policies, the SPEC.md worked examples, replay of
completion logs, and the valid-schedule property (acceptance criterion 4)."""
import json

import pytest

from oracle import oracle as O
from paper_2009_07482_b200 import hetsim, workloads
from paper_2009_07482_b200._native import HetsimError
from tests import dag_gen


def sched(text, params, **kw):
    return hetsim.run_schedule(hetsim.parse_spec(text, params), **kw)


def _times(spec_o, seed):
    return {"gpu": {k: f"{(k * 13 + seed) % 7 + 1}" for k in spec_o.kernels},
            "cpu": {k: f"{(k * 5 + seed) % 11 + 3}/2" for k in spec_o.kernels}}


@pytest.mark.parametrize("seed", range(200))
@pytest.mark.parametrize("policy", ["clustering", "eager", "heft"])
def test_random_dags_match_oracle(seed, policy):
    text, params = dag_gen.layered_dag(seed, cpu_frac=0.25)
    spec_o = O.Spec(text, params)
    cpu = [0] if seed % 3 == 0 else []
    times = _times(spec_o, seed) if seed % 2 else None
    try:
        ours = sched(text, params, policy=policy, times=times, cpu_devices=cpu)
    except HetsimError as e:
        with pytest.raises(O.OracleError) as oe:
            O.schedule(spec_o, policy, times=times, cpu_devices=cpu)
        assert oe.value.errc == e.errc == "Deadlock"
        return
    ref = O.schedule(spec_o, policy, times=times, cpu_devices=cpu)
    assert ours == ref
    _valid_schedule(spec_o, ours)


def _valid_schedule(spec_o, res):
    """Every inter-component edge: the producer's kernel finished before the consumer
    component was dispatched (PAPER.md:200 'dispatched in a topologically sorted fashion')."""
    comp_of = spec_o.comp_of
    dispatch_at = {c: i for i, (c, _) in enumerate(res["dispatches"])}
    assert sorted(dispatch_at) == list(range(len(spec_o.tc)))
    finish_pos = {k: i for i, k in enumerate(res["kernel_finish_order"])}
    assert len(finish_pos) == len(spec_o.kernels)
    for s, _, d, _ in spec_o.edges:
        if comp_of[s] != comp_of[d]:
            assert dispatch_at[comp_of[s]] < dispatch_at[comp_of[d]]
        assert finish_pos[s] < finish_pos[d] or comp_of[s] == comp_of[d]


@pytest.mark.parametrize("seed", range(40))
def test_nonconvex_partitions(seed):
    text, params = dag_gen.layered_dag(2000 + seed, convex=False)
    spec_o = O.Spec(text, params)
    try:
        ours = sched(text, params)
    except HetsimError as e:
        assert e.errc == "Deadlock" and e.exit_code == 1
        with pytest.raises(O.OracleError):
            O.schedule(spec_o)
        return
    assert ours == O.schedule(spec_o)


def test_fig6_callback_semantics():
    """on GPU, r1 completing finishes k3 but not k4; the device returns
    only after every queue's terminal command completed."""
    t, p = workloads.fig6_component()
    log = [[1, 1], [1, 2], [0, 7], [0, 5], [0, 9], [2, 3]]
    res = sched(t, p, replay=log)
    assert res["dispatches"] == [[1, 0], [0, 0], [2, 0]]
    assert res["kernel_finish_order"] == [5, 3, 4, 0, 1, 2, 6]
    assert res == O.schedule(O.Spec(t, p), replay=log)


def test_select_examples():
    # F={T(cpu)}, A={gpu0} -> clustering never selects -> Deadlock
    t, p = workloads.fig7_spec()
    doc = json.loads(t)
    doc["cq"] = [{"device": 0, "queues": 1}]
    with pytest.raises(HetsimError) as e:
        sched(json.dumps(doc), p)
    assert e.value.errc == "Deadlock"
    # eager pairs the top-ranked kernel with the lowest-id device even if it is the CPU
    t, p = workloads.head_dag(1, 64, "per_kernel", queues=1)
    doc = json.loads(t)
    doc["cq"] = [{"device": 0, "queues": 1}, {"device": 1, "queues": 1}]
    res = sched(json.dumps(doc), p, policy="eager", cpu_devices=[0])
    assert res["dispatches"][0][1] == 0
    # heft: t(k,gpu)=5, t(k,cpu)=50 -> gpu
    times = {"gpu": {k: "5" for k in range(8)}, "cpu": {k: "50" for k in range(8)}}
    res = sched(json.dumps(doc), p, policy="heft", cpu_devices=[0], times=times)
    assert res["dispatches"][0][1] == 1


def test_encoder_plan_shapes():
    t, p, _ = workloads.encoder(layers=2)
    res = sched(t, p)
    assert len(res["dispatches"]) == 18
    # heads of layer 1 are ready together and outrank the tail (bottom-level rank)
    assert [c for c, _ in res["dispatches"][:8]] == list(range(8))
    assert res == O.schedule(O.Spec(t, p))
