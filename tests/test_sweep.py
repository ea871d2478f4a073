"""Expt. 1 sweep (SPEC.md sweep_clustering examples) in simulation
with synthetic profiles (SPEC.md DESIGN DECISIONS: GEMM share 0.4, transpose /
softmax share 0.1 on the GPU, so three level-1 GEMMs can overlap)."""
import json

import pytest

from paper_2009_07482_b200 import sweep

GPU = {"gemm": 1.0, "transpose": 0.25, "softmax": 0.25}
SHARE = {"gemm": 0.4, "transpose": 0.1, "softmax": 0.1}
CPU_SLOW = {"gemm": 20.0, "transpose": 2.0, "softmax": 2.0}


def test_grid_is_the_cartesian_product_of_valid_configurations():
    mcs = sweep.configurations(2, q_gpu=range(1, 4), q_cpu=range(1, 3))
    assert len(mcs) == len(set(mcs))
    assert (1, 0, 0) in mcs
    # h_cpu = 0: q_gpu x {0}; 0 < h_cpu < H: q_gpu x q_cpu; h_cpu = H: {0} x q_cpu
    assert len(mcs) == 3 + 3 * 2 + 2
    assert all((c == 0) == (h == 0) for _, c, h in mcs)


def test_head_spec_maps_the_first_heads_to_the_cpu():
    text, params = sweep.head_spec(3, 64, 2, 1, 1)
    doc = json.loads(text)
    per = len(doc["kernels"]) // 3
    assert {k["dev"] for k in doc["kernels"][:per]} == {"cpu"}
    assert {k["dev"] for k in doc["kernels"][per:]} == {"gpu"}
    assert doc["cq"] == [{"device": 0, "queues": 2}, {"device": 1, "queues": 1}]
    with pytest.raises(ValueError):
        sweep.head_spec(2, 64, 1, 0, 1)  # CPU heads without CPU queues


def test_default_configuration_is_fully_serialised():
    """mc = (1,0,0): one in-order GPU queue, so the makespan is the sum of the node times."""
    r = sweep.simulate(1, 256, (1, 0, 0), GPU, CPU_SLOW, SHARE)
    total = 6 * GPU["gemm"] + GPU["transpose"] + GPU["softmax"]  # 8 kernels per head
    assert r["makespan_ms"] == pytest.approx(total, abs=2e-3)


def test_more_gpu_queues_beat_the_default_with_overlapping_gemms():
    t = sweep.sweep_clustering(4, 256, GPU, CPU_SLOW, SHARE, q_gpu=range(1, 6), h_cpu=[0])
    assert t["best"]["mc"][0] >= 2
    assert t["best_vs_default"] > 1.0


def test_all_heads_on_a_slow_cpu_is_worse():
    t = sweep.sweep_clustering(4, 256, GPU, CPU_SLOW, SHARE, q_gpu=[3], q_cpu=[1, 2], h_cpu=[0, 1, 4])
    by = {tuple(r["mc"]): r["makespan_ms"] for r in t["rows"]}
    assert by[(0, 1, 4)] > max(by[(3, 0, 0)], by[(3, 1, 1)])
    csv = sweep.to_csv(t).splitlines()
    assert csv[0].startswith("heads,beta,q_gpu") and len(csv) == 1 + len(t["rows"])


def test_acceptance_5_fine_grained_head_beats_coarse():
    """SPEC acceptance criterion 5 (Figs. 4-5): one whole head on the GPU with the shipped
    overlap profile, makespan(q_gpu = 3) <= 0.95 x makespan(q_gpu = 1)."""
    fine = sweep.simulate(1, 256, (3, 0, 0), GPU, CPU_SLOW, SHARE)["makespan_ms"]
    coarse = sweep.simulate(1, 256, (1, 0, 0), GPU, CPU_SLOW, SHARE)["makespan_ms"]
    assert fine <= 0.95 * coarse


@pytest.mark.parametrize("heads", [4, 8])
def test_acceptance_6_expt1_speedup(heads):
    """SPEC acceptance criterion 6 (Expt. 1): over q_gpu in [1, 5] with h_cpu = 0 the best
    fine-grained configuration is >= 1.10x faster than mc = (1, 0, 0)."""
    t = sweep.sweep_clustering(heads, 256, GPU, CPU_SLOW, SHARE, q_gpu=range(1, 6), h_cpu=[0])
    assert t["best_vs_default"] >= 1.10
