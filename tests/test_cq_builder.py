"""setup_cq / enq / set_dependencies / set_callbacks (the reference ships only
the declarations, cq_builder.hpp:17-79). Pinned by:
  * the paper's Fig. 8 golden (acceptance criterion 2);
  * SPEC.md's per-op examples (:225-227, :234-236, :244-246, :253-255);
  * the structural invariants of SPEC.md:257-262 over >= 200 random layered DAGs
    (acceptance criterion 3);
  * equality with the independent Python restatement in oracle/oracle.py.
"""
import json

import pytest

from oracle import oracle as O
from paper_2009_07482_b200 import hetsim, workloads
from paper_2009_07482_b200._native import HetsimError
from tests import dag_gen


def cq(text, params, comp, queues, device_type="gpu", device=0):
    return hetsim.setup_cq(hetsim.parse_spec(text, params), comp, device, device_type, queues)


def test_fig8_golden():
    t, p = workloads.fig6_component()
    q = cq(t, p, 0, 3)
    assert q["queues"] == [["w1", "w2", "e1", "e4", "r1"], ["w3", "e2", "e5", "r2"], ["e3"]]
    assert q["deps"] == [["e1", "e2"], ["e1", "e3"], ["e2", "e4"], ["e3", "e5"]]
    assert sorted(q["end_marks"]) == ["r1", "r2"]
    assert sorted(q["callbacks"]) == ["e3", "r1", "r2"]      # + terminal command of every queue
    kinds = {c["label"]: c for c in q["commands"]}
    assert kinds["w1"]["dependent"] == 1 and kinds["w2"]["dependent"] == 1   # inter edges (b0,b2), (b1,b3)
    assert kinds["w3"]["dependent"] == 0                                       # isolated write b5


def test_fig8_with_isolated_b8():
    """PAPER.md:169 makes (b8, k2) an isolated write; with it, q2 = [w4, e3] (SURVEY §8c ambiguity 1)."""
    t, p = workloads.fig6_component(with_b8=True)
    q = cq(t, p, 0, 3)
    assert q["queues"][2] == ["w4", "e3"]


def test_fig8_cpu_callbacks():
    t, p = workloads.fig6_component()
    q = cq(t, p, 0, 3, device_type="cpu")
    assert sorted(q["end_marks"]) == ["e4", "e5"]


def test_spec_examples_single_queue_and_singleton():
    t, p = workloads.fig6_component()
    q = cq(t, p, 0, 1)
    assert q["deps"] == []  # all commands in one queue -> deps = {}
    q = cq(t, p, 1, 1)      # singleton producer component k5: ndrange + dependent reads
    assert q["queues"] == [["e1", "r1", "r2"]]
    q = cq(t, p, 2, 1)      # consumer k6: two dependent writes, ndrange, isolated read
    assert q["queues"] == [["w1", "w2", "e1", "r1"]]


def test_transformer_head_round_robin():
    """8-kernel head, r=3: level-1 GEMMs land in distinct queues."""
    t, p = workloads.head_dag(1, 256)
    q = cq(t, p, 0, 3)
    nd = [c for c in q["commands"] if c["kind"] == "ndrange"]
    assert len(nd) == 8
    assert {c["queue"] for c in nd[:3]} == {0, 1, 2}


def test_already_processed_and_errors():
    t, p = workloads.fig6_component()
    with pytest.raises(HetsimError) as e:
        cq(t, p, 0, 0)
    assert e.value.errc == "InvalidParam"


def _audit(q, spec, comp):
    """SPEC.md:257-262 invariants on one structure."""
    cmds = q["commands"]
    front, end = comp["front"], comp["end"]
    kinds = O.edge_kinds(spec)
    pos = {}
    for qi, lst in enumerate(q["queues"]):
        for i, lab in enumerate(lst):
            pos[lab] = (qi, i)
    by_label = {c["label"]: c for c in cmds}
    # deps are cross-queue and point forward in enqueue order
    for a, b in q["deps"]:
        assert pos[a][0] != pos[b][0]
        assert by_label[a]["event"] < by_label[b]["event"]
    for k in comp["kernels"]:
        mine = [c for c in cmds if c["kernel"] == k]
        nds = [c for c in mine if c["kind"] == "ndrange"]
        assert len(nds) == 1                       # exactly one ndrange per kernel
        ndq, ndi = pos[nds[0]["label"]]
        for c in mine:                              # writes before, reads after, same queue
            qi, i = pos[c["label"]]
            assert qi == ndq
            if c["kind"] == "write":
                assert i < ndi
            if c["kind"] == "read":
                assert i > ndi
        dep_w = [c for c in mine if c["kind"] == "write" and c["dependent"]]
        dep_r = [c for c in mine if c["kind"] == "read" and c["dependent"]]
        inter_in = [ei for ei, e in enumerate(spec.edges) if e[2] == k and kinds[ei] == "inter"]
        inter_out = [ei for ei, e in enumerate(spec.edges) if e[0] == k and kinds[ei] == "inter"]
        # redundancy elimination and exact counts
        assert len(dep_w) == (len(inter_in) if k in front else 0)
        assert len(dep_r) == (len(inter_out) if k in end else 0)
    terminals = {lst[-1] for lst in q["queues"] if lst}
    assert terminals <= set(q["callbacks"])


@pytest.mark.parametrize("seed", range(220))
def test_random_structures_match_oracle_and_invariants(seed):
    text, params = dag_gen.layered_dag(seed)
    spec_o = O.Spec(text, params)
    spec = hetsim.parse_spec(text, params)
    comps = O.components(spec_o)
    for comp in comps:
        for r in (1, 2, 3, 5):
            for dt in ("gpu", "cpu"):
                ours = hetsim.setup_cq(spec, comp["id"], 0, dt, r)
                ref = O.setup_cq(spec_o, comp["id"], 0, dt, r)
                for key in ("queues", "deps", "callbacks", "end_marks"):
                    assert ours[key] == ref[key], (seed, comp["id"], r, dt, key)
                assert [{k: v for k, v in c.items()} for c in ours["commands"]] == ref["commands"]
                _audit(ours, spec_o, comp)


def test_determinism():
    t, p, _ = workloads.encoder(layers=2)
    a = cq(t, p, 8, 3)
    b = cq(t, p, 8, 3)
    assert json.dumps(a) == json.dumps(b)
