"""roofline.dag_bound against the per-config bounds SURVEY.md §8d states (computed there
by hand from the same per-node work model, P = 276 TFLOP/s, B = 6543.1 GB/s)."""
import pytest

from paper_2009_07482_b200 import roofline, workloads

P, B = 276.0, 6543.1


def _enc(layers, n):
    text, params, meta = workloads.encoder(layers=layers)
    shared = [(w["kernel"], w["pos"]) for w in meta["weights"]]
    return roofline.dag_bound(text, params, n, P, B, shared_inputs=shared, io_bytes=2 * 128 * 512 * 4)


def test_small_configs_are_critical_path_bound():
    text, params = workloads.fork_join()
    c1 = roofline.dag_bound(text, params, 1, P, B)
    assert c1["bound"] == "critical_path"
    assert c1["t_star_ms"] * 1e3 == pytest.approx(0.363, abs=1e-3)  # µs
    text, params = workloads.attention()
    c2 = roofline.dag_bound(text, params, 1, P, B)
    assert c2["t_star_ms"] * 1e3 == pytest.approx(0.080, abs=1e-3)


@pytest.mark.parametrize("layers,n,cp_us,t_star_ms", [(1, 1, 2.41, 2.83e-3), (6, 64, 14.5, 1.087), (12, 4096, 29.0, 139.1)])
def test_encoder_bounds_match_survey(layers, n, cp_us, t_star_ms):
    r = _enc(layers, n)
    assert r["critical_path_ms"] * 1e3 == pytest.approx(cp_us, rel=5e-3)
    assert r["t_star_ms"] == pytest.approx(t_star_ms, rel=5e-3)
    assert r["bound"] == "tensor"


def test_node_work_conventions():
    k = {"name": "gemm", "varArguments": [{"pos": 3, "value": "128"}, {"pos": 4, "value": "64"},
                                          {"pos": 5, "value": "512"}]}
    f, b = roofline.node_work(k, {})
    assert f == 2 * 128 * 64 * 512 and b == 4 * (128 * 512 + 512 * 64 + 128 * 64)
    k = {"name": "softmax", "inputBuffers": [{"pos": 0, "size": "S*S"}], "outputBuffers": [{"pos": 1, "size": "S*S"}],
         "varArguments": []}
    assert roofline.node_work(k, {"S": 128}) == (0.0, 8.0 * 128 * 128)
