"""Sanity of the CPU oracle itself: its node kernels against float64 numpy,
its expression evaluator against the reference's compiled one, and its DAG
executor against a direct numpy evaluation of the encoder layer math."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2009_07482_b200 import workloads


def test_gemm_kernel_vs_float64(oracle_mod):
    rng = np.random.default_rng(0)
    for (M, N, K, nt) in [(17, 33, 65, 0), (128, 64, 512, 0), (40, 24, 8, 1)]:
        A = rng.standard_normal((2, M * K)).astype(np.float32)
        B = rng.standard_normal((N * K,)).astype(np.float32)
        C = np.empty((2, M * N), np.float32)
        oracle_mod.run_node("gemm_nt" if nt else "gemm", [A, B], [M * K, 0], C, M * N, [M, N, K], 2)
        Bm = B.reshape(N, K).T if nt else B.reshape(K, N)
        for b in range(2):
            ref = A[b].reshape(M, K).astype(np.float64) @ Bm.astype(np.float64)
            assert np.max(np.abs(C[b].reshape(M, N) - ref)) / np.max(np.abs(ref)) < 1e-5


def test_exact_kernels(oracle_mod):
    x = workloads.uniform(3, 1, 128 * 64).reshape(1, -1)
    out = np.empty_like(x)
    oracle_mod.run_node("transpose", [x], [x.size], out, x.size, [128, 64], 1)
    assert np.array_equal(out.reshape(64, 128), x.reshape(128, 64).T)
    oracle_mod.run_node("scale", [x], [x.size], out, x.size, [x.size, 1, 8], 1)
    assert np.array_equal(out, x * np.float32(0.125))


def test_softmax_and_layernorm_vs_numpy(oracle_mod):
    x = workloads.uniform(4, 2, 128 * 128).reshape(1, -1) * 3
    out = np.empty_like(x)
    oracle_mod.run_node("softmax", [x], [x.size], out, x.size, [128, 128, 1, 8], 1)
    z = x.reshape(128, 128).astype(np.float64) / 8
    ref = np.exp(z - z.max(1, keepdims=True))
    ref /= ref.sum(1, keepdims=True)
    assert np.max(np.abs(out.reshape(128, 128) - ref)) < 1e-6
    a, b = workloads.uniform(5, 3, 4 * 512).reshape(1, -1), workloads.uniform(6, 3, 4 * 512).reshape(1, -1)
    g, be = np.ones(512, np.float32), np.zeros(512, np.float32)
    oracle_mod.run_node("add_layernorm", [a, b, g, be], [a.size, a.size, 0, 0], out[:, :a.size], a.size, [4, 512], 1)
    v = (a + b).reshape(4, 512).astype(np.float64)
    ref = (v - v.mean(1, keepdims=True)) / np.sqrt(v.var(1, keepdims=True) + 1e-5)
    assert np.max(np.abs(out[0, :a.size].reshape(4, 512) - ref)) < 1e-5


@pytest.mark.parametrize("expr", ["M*N", "M/2", "7/2", "N/0", "(M+1)*(N-1)", "-M*-N", "M*", "X", "12/4/3"])
def test_expr_evaluator_matches_reference(expr):
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    ref = O.ref_query({"op": "expr", "expr": expr, "params": {"M": 4, "N": 6}})
    try:
        v = O.eval_expr(expr, {"M": 4, "N": 6})
        assert ref["ok"] and ref["value"] == v
    except O.OracleError as e:
        assert not ref["ok"] and ref["errc"] == e.errc


def test_dag_executor_matches_layer_math(oracle_mod):
    """One encoder layer through the oracle DAG executor == the same math in numpy float64."""
    text, params, meta = workloads.encoder(layers=1)
    x = workloads.encoder_inputs(meta, params, 1).reshape(1, -1)
    arrays = {(i["kernel"], i["pos"]): x for i in meta["x_inputs"]}
    W = workloads.encoder_weights(meta)
    for k, w in W.items():
        arrays[k] = w.reshape(-1)
    out = oracle_mod.run_dag(text, params, arrays, 1)
    y = out[(meta["output"]["kernel"], meta["output"]["pos"])].reshape(128, 512).astype(np.float64)
    X = x.reshape(128, 512).astype(np.float64)
    ws = [w for w in meta["weights"]]
    get = lambda i: W[(ws[i]["kernel"], ws[i]["pos"])].astype(np.float64)  # noqa: E731
    Z = []
    for h in range(8):
        q, k, v, wh = (get(4 * h + j) for j in range(4))
        Q, K, V = X @ q, X @ k, X @ v
        A = Q @ K.T / 8
        P = np.exp(A - A.max(1, keepdims=True))
        P /= P.sum(1, keepdims=True)
        Z.append(P @ V @ wh)
    cat = np.concatenate(Z, axis=1)

    def ln(v, g, b):
        return (v - v.mean(1, keepdims=True)) / np.sqrt(v.var(1, keepdims=True) + 1e-5) * g + b
    g1, b1, w1, w2, g2, b2 = (get(32 + j) for j in range(6))
    h1 = ln(X + cat, g1, b1)
    f = np.maximum(h1 @ w1, 0) @ w2
    ref = ln(h1 + f, g2, b2)
    assert np.max(np.abs(y - ref)) / np.max(np.abs(ref)) < 1e-5


def test_attn_head_node_is_the_head_chain():
    """The oracle's attn_head node is defined as the paper's head chain: a layer
    written with fused heads gives bit-identical outputs to the 8-kernel heads
    (same inputs and the same weights, matched by role)."""
    from oracle import oracle as O
    from paper_2009_07482_b200 import workloads
    text0, params, meta0 = workloads.encoder(layers=1)
    w0 = workloads.encoder_weights(meta0)
    by_role = {m["key"]: w0[(m["kernel"], m["pos"])] for m in meta0["weights"]}
    outs = []
    for fused in (False, True):
        text, params, meta = workloads.encoder(layers=1, fused_heads=fused)
        x = workloads.encoder_inputs(meta, params, 2).reshape(2, -1)
        arrays = {(i["kernel"], i["pos"]): x for i in meta["x_inputs"]}
        for m in meta["weights"]:
            arrays[(m["kernel"], m["pos"])] = by_role[m["key"]].reshape(-1)
        out = O.run_dag(text, params, arrays, 2)
        outs.append(out[(meta["output"]["kernel"], meta["output"]["pos"])])
    assert np.array_equal(outs[0], outs[1])
