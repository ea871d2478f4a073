"""Per-operator parity on the B200: sm_100a kernels (through hs_launch) vs the
CPU oracle (oracle/kernels.c) on identical seeded inputs.

Tolerances (north_star): GEMM in 3xTF32 mode <= 1e-4 normwise relative error
per output; transpose / concat / scale-by-1/8 / add are bit-exact; softmax and
add+LayerNorm differ from the sequential oracle only by summation order
(<= 1e-5 normwise).
"""
import numpy as np
import pytest

from paper_2009_07482_b200.workloads import uniform

pytestmark = pytest.mark.gpu

TOL_TF32X3 = 1e-4


def _t(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _rand(uid, shape, seed=11):
    n = int(np.prod(shape))
    return uniform(seed, uid, n).reshape(shape)


GEMM_CASES = [
    # (M, N, K, op, batch, shared_B)
    (256, 256, 256, "gemm", 1, False),      # C1 fork-join
    (128, 64, 512, "gemm", 4, True),        # C3 Q/K/V projection (shared weight)
    (128, 128, 64, "gemm", 3, False),       # C3 QK^T via transpose
    (128, 128, 64, "gemm_nt", 2, False),    # C2 QK^T
    (128, 64, 128, "gemm", 2, False),       # PV
    (128, 64, 64, "gemm", 2, True),         # C W_h
    (128, 2048, 512, "gemm_relu", 2, True),  # FFN1
    (128, 512, 2048, "gemm", 2, True),      # FFN2
    (100, 72, 36, "gemm", 2, False),        # ragged M/N/K tails
    (130, 200, 44, "gemm_nt", 1, False),
    (64, 8, 4, "gemm", 1, False),
    # single-instance launches with a long K loop run split-K: a cluster of CTAs per
    # output tile, partials reduced over DSMEM (ReLU after the sum), ragged tails
    (128, 512, 2048, "gemm", 1, True),
    (256, 256, 256, "gemm", 1, False),
    (100, 64, 1000, "gemm_nt", 1, False),
    (128, 2048, 512, "gemm_relu", 1, True),
    (100, 72, 1000, "gemm", 1, False),
    (200, 130, 600, "gemm_relu", 1, False),
]


@pytest.mark.parametrize("M,N,K,op,shared", [(256, 256, 256, "gemm", False), (128, 2048, 512, "gemm_relu", True),
                                             (128, 512, 2048, "gemm", True)])
def test_single_instance_split_k_is_bit_reproducible(M, N, K, op, shared):
    """Cluster split-K reduces the K-split partials in rank order over DSMEM: the same
    launch gives bit-identical outputs every time (no atomics)."""
    from tests.gpu_util import launch
    import torch
    A = _t(_rand(41, (1, M * K)))
    B = _t((_rand(42, (N * K,) if shared else (1, N * K)) * np.float32(1.0 / np.sqrt(K))).astype(np.float32))
    outs = []
    for _ in range(3):
        out = torch.full((1, M * N), float("nan"), device="cuda")
        launch(op, [A, B], out, [M, N, K], batch=1)
        outs.append(out.cpu().numpy())
    assert np.isfinite(outs[0]).all()
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])


@pytest.mark.parametrize("M,N,K,op,batch,shared", GEMM_CASES)
@pytest.mark.parametrize("math", ["tf32x3", "simt"])
def test_gemm_parity(M, N, K, op, batch, shared, math, oracle_mod):
    from tests.gpu_util import launch, normwise
    import torch
    A = _rand(1, (batch, M * K))
    Bshape = (N * K,) if shared else (batch, N * K)
    B = _rand(2, Bshape) * np.float32(1.0 / np.sqrt(K))
    ref = np.empty((batch, M * N), np.float32)
    oracle_mod.run_node(op, [A, B.astype(np.float32)], [M * K, 0 if shared else N * K], ref, M * N, [M, N, K], batch)
    out = torch.full((batch, M * N), float("nan"), device="cuda")
    launch(op, [_t(A), _t(B.astype(np.float32))], out, [M, N, K], math=math, batch=batch)
    y = out.cpu().numpy()
    assert np.isfinite(y).all()
    for b in range(batch):
        err = normwise(y[b], ref[b])
        assert err <= (TOL_TF32X3 if math == "tf32x3" else 1e-5), (b, err)


PAIR_CASES = [  # CTA-pair path (resident B, N >= 192, >= 2 row blocks): odd row-block tails, m-tiles, ragged N
    (128, 2048, 512, "gemm_relu", 3, True), (200, 256, 96, "gemm", 3, True), (130, 512, 64, "gemm", 1, True),
    (128, 300, 64, "gemm_nt", 2, True), (128, 192, 512, "gemm", 5, True)]


@pytest.mark.parametrize("M,N,K,op,batch,shared", [c for c in GEMM_CASES if c[5]] + [(128, 128, 64, "gemm_nt", 3, True),
                                                                              (72, 100, 36, "gemm", 2, True)]
                         + PAIR_CASES)
@pytest.mark.parametrize("math", ["tf32x3", "tf32", "bf16x3"])
def test_gemm_presplit_weights(M, N, K, op, batch, shared, math, oracle_mod):
    """Resident-weight path: B pre-split once into K-major tf32 (or bf16) planes, fed by TMA."""
    from tests.gpu_util import launch, normwise, split_weights
    import torch
    A = _rand(31, (batch, M * K))
    B = (_rand(32, (N * K,)) * np.float32(1.0 / np.sqrt(K))).astype(np.float32)
    ref = np.empty((batch, M * N), np.float32)
    oracle_mod.run_node(op, [A, B], [M * K, 0], ref, M * N, [M, N, K], batch)
    Bt = _t(B)
    planes = split_weights(Bt, op == "gemm_nt", N, K, bf16=math == "bf16x3")
    out = torch.full((batch, M * N), float("nan"), device="cuda")
    launch(op, [_t(A), Bt], out, [M, N, K], math=math, batch=batch, aux=planes)
    y = out.cpu().numpy()
    tol = {"tf32x3": TOL_TF32X3, "bf16x3": 5e-5, "tf32": 5e-3}[math]
    for b in range(batch):
        assert normwise(y[b], ref[b]) <= tol, b


def test_gemm_tf32_single_term_is_coarser(oracle_mod):
    """The 1-term TF32 mode is visibly less accurate than 3xTF32 (sanity of the split)."""
    from tests.gpu_util import launch, normwise
    import torch
    M, N, K = 128, 128, 2048
    A, B = _rand(3, (1, M * K)), _rand(4, (1, K * N))
    ref = np.empty((1, M * N), np.float32)
    oracle_mod.run_node("gemm", [A, B], [M * K, K * N], ref, M * N, [M, N, K], 1)
    errs = {}
    for math in ("tf32", "tf32x3"):
        out = torch.empty((1, M * N), device="cuda")
        launch("gemm", [_t(A), _t(B)], out, [M, N, K], math=math)
        errs[math] = normwise(out.cpu().numpy(), ref)
    assert errs["tf32x3"] <= TOL_TF32X3
    assert errs["tf32x3"] * 10 < errs["tf32"], errs


@pytest.mark.parametrize("math,presplit", [("tf32x3", False), ("tf32x3", True), ("bf16x3", True), ("simt", False)])
def test_gemm_writes_column_block(math, presplit, oracle_mod):
    """out_ld: a GEMM writes its [M,N] result as columns [off, off+N) of a wider
    row-major matrix (how a concat input is produced in place); the other
    columns are untouched."""
    from tests.gpu_util import launch, normwise, split_weights
    import torch
    M, N, K, batch, width, off = 128, 64, 64, 3, 512, 192
    A = _rand(41, (batch, M * K))
    B = (_rand(42, (N * K,)) * np.float32(1.0 / np.sqrt(K))).astype(np.float32)
    ref = np.empty((batch, M * N), np.float32)
    oracle_mod.run_node("gemm", [A, B], [M * K, 0], ref, M * N, [M, N, K], batch)
    Bt = _t(B)
    planes = split_weights(Bt, False, N, K, bf16=math == "bf16x3") if presplit else None
    Y = torch.full((batch, M * width), -7.0, device="cuda")
    launch("gemm", [_t(A), Bt], Y, [M, N, K], math=math, batch=batch, aux=planes, out_ld=width, out_offset=off)
    y = Y.cpu().numpy().reshape(batch, M, width)
    tol = {"tf32x3": TOL_TF32X3, "bf16x3": 5e-5, "simt": 1e-5}[math]
    for b in range(batch):
        assert normwise(y[b, :, off:off + N].reshape(-1), ref[b]) <= tol, b
    mask = np.ones(width, bool)
    mask[off:off + N] = False
    assert (y[:, :, mask] == -7.0).all()


@pytest.mark.parametrize("M,N,K,op,batch", [(128, 128, 64, "gemm_nt", 3), (128, 128, 64, "gemm", 2),
                                             (100, 72, 36, "gemm_nt", 2), (200, 128, 64, "gemm", 1)])
@pytest.mark.parametrize("math", ["tf32x3", "tf32"])
def test_gemm_softmax_epilogue(M, N, K, op, batch, math, oracle_mod):
    """HS_EPI_SOFTMAX: P = softmax_row((A·B)·s) from one launch, against the oracle's
    gemm followed by its softmax (the GEMM's own error passes through exp)."""
    from tests.gpu_util import launch, normwise
    import torch
    A = _rand(51, (batch, M * K)) * np.float32(2)
    B = _rand(52, (batch, N * K))
    S = np.empty((batch, M * N), np.float32)
    oracle_mod.run_node(op, [A, B], [M * K, N * K], S, M * N, [M, N, K], batch)
    ref = np.empty_like(S)
    oracle_mod.run_node("softmax", [S], [M * N], ref, M * N, [M, N, 1, 8], batch)
    out = torch.full((batch, M * N), float("nan"), device="cuda")
    launch(op, [_t(A), _t(B)], out, [M, N, K], fparam=(0.125, 1e-5), math=math, batch=batch, epilogue=1)
    y = out.cpu().numpy()
    assert np.isfinite(y).all()
    assert np.allclose(y.reshape(-1, N).sum(axis=1), 1.0, atol=1e-5)
    tol = TOL_TF32X3 if math == "tf32x3" else 5e-3
    for b in range(batch):
        assert normwise(y[b], ref[b]) <= tol, b


def test_softmax_epilogue_rejects_wide_rows():
    from paper_2009_07482_b200._native import HetsimError
    from tests.gpu_util import launch
    import torch
    A = torch.zeros(1, 128 * 64, device="cuda")
    B = torch.zeros(1, 256 * 64, device="cuda")
    out = torch.empty(1, 128 * 256, device="cuda")
    with pytest.raises(HetsimError):
        launch("gemm_nt", [A, B], out, [128, 256, 64], epilogue=1)


@pytest.mark.parametrize("R,C,batch", [(128, 64, 3), (64, 128, 1), (37, 45, 2)])
def test_transpose_bit_exact(R, C, batch, oracle_mod):
    from tests.gpu_util import launch
    import torch
    A = _rand(5, (batch, R * C))
    ref = np.empty_like(A)
    oracle_mod.run_node("transpose", [A], [R * C], ref, R * C, [R, C], batch)
    out = torch.empty((batch, R * C), device="cuda")
    launch("transpose", [_t(A)], out, [R, C], batch=batch)
    assert np.array_equal(out.cpu().numpy(), ref)


@pytest.mark.parametrize("n,batch", [(128 * 128, 2), (1001, 3)])
def test_scale_and_add_bit_exact(n, batch, oracle_mod):
    from tests.gpu_util import launch
    import torch
    A, B = _rand(6, (batch, n)), _rand(7, (batch, n))
    ref = np.empty_like(A)
    oracle_mod.run_node("scale", [A], [n], ref, n, [n, 1, 8], batch)
    out = torch.empty((batch, n), device="cuda")
    launch("scale", [_t(A)], out, [n], fparam=(0.125, 1e-5), batch=batch)
    assert np.array_equal(out.cpu().numpy(), ref)
    oracle_mod.run_node("add", [A, B], [n, n], ref, n, [n], batch)
    launch("add", [_t(A), _t(B)], out, [n], batch=batch)
    assert np.array_equal(out.cpu().numpy(), ref)


@pytest.mark.parametrize("rows,cols,batch,num,den", [(128, 128, 3, 1, 8), (128, 512, 1, 1, 1), (17, 100, 2, 1, 1)])
def test_softmax(rows, cols, batch, num, den, oracle_mod):
    from tests.gpu_util import launch, normwise
    import torch
    A = _rand(8, (batch, rows * cols)) * np.float32(4)
    ref = np.empty_like(A)
    oracle_mod.run_node("softmax", [A], [rows * cols], ref, rows * cols, [rows, cols, num, den], batch)
    out = torch.empty((batch, rows * cols), device="cuda")
    launch("softmax", [_t(A)], out, [rows, cols], fparam=(num / den, 1e-5), batch=batch)
    y = out.cpu().numpy()
    assert normwise(y, ref) <= 1e-5
    assert np.allclose(y.reshape(-1, cols).sum(axis=1), 1.0, atol=1e-5)


@pytest.mark.parametrize("rows,cols,batch", [(128, 512, 2), (9, 96, 3)])
def test_add_layernorm(rows, cols, batch, oracle_mod):
    from tests.gpu_util import launch, normwise
    import torch
    A, B = _rand(9, (batch, rows * cols)), _rand(10, (batch, rows * cols))
    g = (1 + 0.1 * _rand(12, (cols,))).astype(np.float32)
    be = (0.1 * _rand(13, (cols,))).astype(np.float32)
    ref = np.empty_like(A)
    oracle_mod.run_node("add_layernorm", [A, B, g, be], [rows * cols, rows * cols, 0, 0], ref, rows * cols,
                        [rows, cols], batch)
    out = torch.empty((batch, rows * cols), device="cuda")
    launch("add_layernorm", [_t(A), _t(B), _t(g), _t(be)], out, [rows, cols], fparam=(1.0, 1e-5), batch=batch)
    assert normwise(out.cpu().numpy(), ref) <= 1e-5


@pytest.mark.parametrize("count,rows,cols,batch", [(8, 128, 64, 2), (3, 5, 7, 2)])
def test_concat_bit_exact(count, rows, cols, batch, oracle_mod):
    from tests.gpu_util import launch
    import torch
    Z = [_rand(20 + i, (batch, rows * cols)) for i in range(count)]
    ref = np.empty((batch, rows * cols * count), np.float32)
    oracle_mod.run_node("concat", Z, [rows * cols] * count, ref, rows * cols * count, [rows, cols], batch)
    out = torch.empty((batch, rows * cols * count), device="cuda")
    launch("concat", [_t(z) for z in Z], out, [rows, cols], batch=batch)
    assert np.array_equal(out.cpu().numpy(), ref)


def _attn_ref(oracle_mod, Q, K, V, W, S, batch, scale_den=8):
    dk, dw = 64, 64
    A = np.empty((batch, S * S), np.float32)
    oracle_mod.run_node("gemm_nt", [Q, K], [S * dk, S * dk], A, S * S, [S, S, dk], batch)
    P = np.empty_like(A)
    oracle_mod.run_node("softmax", [A], [S * S], P, S * S, [S, S, 1, scale_den], batch)
    C = np.empty((batch, S * dk), np.float32)
    oracle_mod.run_node("gemm", [P, V], [S * S, S * dk], C, S * dk, [S, dk, S], batch)
    Z = np.empty((batch, S * dw), np.float32)
    oracle_mod.run_node("gemm", [C, W], [S * dk, 0], Z, S * dw, [S, dw, dk], batch)
    return Z


@pytest.mark.parametrize("S,batch,math,ld", [(128, 3, "tf32x3", 0), (100, 2, "tf32x3", 0), (128, 5, "tf32", 0),
                                              (128, 3, "tf32x3", 512), (128, 300, "tf32x3", 0)])
def test_attn_head_matches_oracle(S, batch, math, ld, oracle_mod):
    """HS_OP_ATTN_HEAD: Z = softmax(Q Kᵀ/8) V W in one launch, against the oracle's
    four-node chain (gemm_nt, softmax, gemm, gemm)."""
    from tests.gpu_util import launch, normwise, split_weights
    import torch
    dk = 64
    Q, K, V = (_rand(60 + i, (batch, S * dk)) for i in range(3))
    W = (_rand(63, (dk * dk,)) * np.float32(1 / 8)).astype(np.float32)
    ref = _attn_ref(oracle_mod, Q, K, V, W, S, batch)
    Wt = _t(W)
    planes = split_weights(Wt, False, dk, dk)
    width, off = (ld, 128) if ld else (dk, 0)
    Y = torch.full((batch, S * width), -3.0, device="cuda")
    launch("attn_head", [_t(Q), _t(K), _t(V), Wt], Y, [S, dk, dk], fparam=(0.125, 1e-5), math=math, batch=batch,
           aux=planes, out_ld=ld, out_offset=off)
    y = Y.cpu().numpy().reshape(batch, S, width)
    tol = TOL_TF32X3 if math == "tf32x3" else 5e-3
    for b in range(batch):
        assert normwise(y[b, :, off:off + dk].reshape(-1), ref[b]) <= tol, b
    if ld:
        mask = np.ones(width, bool)
        mask[off:off + dk] = False
        assert (y[:, :, mask] == -3.0).all()


def test_attn_head_bit_identical_to_unfused_chain():
    """The fused head keeps every intermediate in TMEM / smem but computes it
    exactly as the unfused tcgen05 chain does (same splits, same MMA order):
    Z is bit-identical to gemm_nt+softmax epilogue -> gemm -> gemm (pre-split W)."""
    from tests.gpu_util import launch, split_weights
    import torch
    S, dk, batch = 128, 64, 4
    Q, K, V = (_t(_rand(70 + i, (batch, S * dk))) for i in range(3))
    W = _t((_rand(73, (dk * dk,)) * np.float32(1 / 8)).astype(np.float32))
    planes = split_weights(W, False, dk, dk)
    P = torch.empty(batch, S * S, device="cuda")
    launch("gemm_nt", [Q, K], P, [S, S, dk], fparam=(0.125, 1e-5), batch=batch, epilogue=1)
    C = torch.empty(batch, S * dk, device="cuda")
    launch("gemm", [P, V], C, [S, dk, S], batch=batch)
    Z0 = torch.empty(batch, S * dk, device="cuda")
    launch("gemm", [C, W], Z0, [S, dk, dk], batch=batch, aux=planes)
    Z1 = torch.empty(batch, S * dk, device="cuda")
    launch("attn_head", [Q, K, V, W], Z1, [S, dk, dk], fparam=(0.125, 1e-5), batch=batch, aux=planes)
    assert torch.equal(Z0, Z1)


def _head_launch(X, planes_qkv, planes_h, Z, S, D, batch, math="tf32x3", ld=0, off=0):
    """HS_OP_HEAD through the C ABI: in = {X, Wh planes}, aux = Wq|Wk|Wv planes."""
    import ctypes
    import torch
    from paper_2009_07482_b200 import _native
    from tests.gpu_util import MATH, stream
    torch.cuda.synchronize()
    L = _native.lib()
    a = _native.OpArgs()
    a.n_in = 2
    a.in_[0], a.in_stride[0] = X.data_ptr(), S * D
    a.in_[1], a.in_stride[1] = planes_h.data_ptr(), 0
    a.aux = planes_qkv.data_ptr()
    a.out, a.out_stride, a.out_ld = Z.data_ptr() + 4 * off, Z.shape[-1], ld
    a.dims[0], a.dims[1], a.dims[2] = S, D, 64
    a.fparam[0] = 0.125
    _native.check(L.hs_launch(stream(), 10, ctypes.byref(a), MATH[math], batch), "hs_launch(head)")
    _native.check(L.hs_stream_sync(stream()), "sync")


def _qkv_planes(Ws, D):
    import torch
    from paper_2009_07482_b200 import _native
    from tests.gpu_util import stream
    planes = torch.empty(2 * 3 * 64 * D, device="cuda")
    torch.cuda.synchronize()
    L = _native.lib()
    for m, W in enumerate(Ws):
        _native.check(L.hs_gemm_split_weights_strided(stream(), W.data_ptr(), 0, 64, D,
                                                      planes.data_ptr() + 4 * m * 64 * D, 3 * 64 * D))
    _native.check(L.hs_stream_sync(stream()))
    return planes


def _grouped_qkv(X, Ws, planes, outs, S, D, batch):
    import ctypes
    import torch
    from paper_2009_07482_b200 import _native
    from tests.gpu_util import stream
    torch.cuda.synchronize()
    L = _native.lib()
    a = _native.OpArgs()
    a.n_in = 2
    a.in_[0], a.in_stride[0] = X.data_ptr(), S * D
    a.in_[1], a.in_stride[1] = Ws[0].data_ptr(), 0
    a.out, a.out_stride = outs[0].data_ptr(), S * 64
    a.dims[0], a.dims[1], a.dims[2] = S, 64, D
    a.aux = planes.data_ptr()
    a.n_out = 3
    for m in range(3):
        a.outs[m], a.out_strides[m] = outs[m].data_ptr(), S * 64
    _native.check(L.hs_launch(stream(), 0, ctypes.byref(a), 0, batch), "hs_launch(grouped qkv)")
    _native.check(L.hs_stream_sync(stream()), "sync")


@pytest.mark.parametrize("S,batch,D", [(128, 1, 512), (128, 4, 512), (128, 7, 512), (100, 3, 512), (128, 300, 512),
                                       (128, 5, 256), (128, 3, 96), (64, 9, 1024), (128, 149, 512), (128, 445, 512)])
def test_head_fused_matches_grouped_qkv_and_attn_head(S, batch, D, oracle_mod):
    """HS_OP_HEAD (projection + attention of two instances in flight per SM, Q/K/V
    never leave the SM) against the two launches it replaces — the grouped Q/K/V
    GEMM writing Q, K, V to HBM, then the fused attention head — and, on sampled
    instances (first, last, and both sides of the 148-CTA wrap), the CPU oracle.
    The P·V terms are accumulated in another order, so the two agree to fp32
    rounding, not bit for bit."""
    from tests.gpu_util import launch, normwise, split_weights
    import torch
    X = _t(_rand(80, (batch, S * D)))
    Ws = [_t((_rand(81 + m, (D * 64,)) * np.float32(1 / np.sqrt(D))).astype(np.float32)) for m in range(3)]
    Wh = _t((_rand(84, (64 * 64,)) * np.float32(1 / 8)).astype(np.float32))
    pq = _qkv_planes(Ws, D)
    ph = split_weights(Wh, False, 64, 64)
    Q, K, V = (torch.empty(batch, S * 64, device="cuda") for _ in range(3))
    _grouped_qkv(X, Ws, pq, (Q, K, V), S, D, batch)
    Z0 = torch.empty(batch, S * 64, device="cuda")
    launch("attn_head", [Q, K, V, Wh], Z0, [S, 64, 64], fparam=(0.125, 1e-5), batch=batch, aux=ph)
    Z1 = torch.full((batch, S * 64), -7.0, device="cuda")
    _head_launch(X, pq, ph, Z1, S, D, batch)
    z0, z1 = Z0.cpu().numpy(), Z1.cpu().numpy()
    for b in range(batch):
        assert normwise(z1[b], z0[b]) <= 1e-5, b
    idx = sorted({0, batch - 1, min(batch - 1, 147), min(batch - 1, 148)})
    x = X.cpu().numpy()[idx]
    proj = []
    for W in Ws:
        out = np.empty((len(idx), S * 64), np.float32)
        oracle_mod.run_node("gemm", [x, W.cpu().numpy()], [S * D, 0], out, S * 64, [S, 64, D], len(idx))
        proj.append(out)
    ref = _attn_ref(oracle_mod, proj[0], proj[1], proj[2], Wh.cpu().numpy(), S, len(idx))
    for j, b in enumerate(idx):
        assert normwise(z1[b], ref[j]) <= TOL_TF32X3, b


@pytest.mark.parametrize("math,ld", [("tf32x3", 0), ("tf32x3", 512), ("tf32", 0)])
def test_head_fused_matches_oracle(math, ld, oracle_mod):
    """HS_OP_HEAD against the oracle's head chain: three projection GEMMs, then
    gemm_nt -> softmax(1/8) -> gemm -> gemm."""
    from tests.gpu_util import normwise, split_weights
    import torch
    S, D, dk, batch = 128, 512, 64, 5
    X = _rand(90, (batch, S * D))
    Ws = [(_rand(91 + m, (D * dk,)) * np.float32(1 / np.sqrt(D))).astype(np.float32) for m in range(3)]
    Wh = (_rand(94, (dk * dk,)) * np.float32(1 / 8)).astype(np.float32)
    proj = []
    for W in Ws:
        out = np.empty((batch, S * dk), np.float32)
        oracle_mod.run_node("gemm", [X, W], [S * D, 0], out, S * dk, [S, dk, D], batch)
        proj.append(out)
    ref = _attn_ref(oracle_mod, proj[0], proj[1], proj[2], Wh, S, batch)
    pq = _qkv_planes([_t(W) for W in Ws], D)
    ph = split_weights(_t(Wh), False, dk, dk)
    width, off = (ld, 128) if ld else (dk, 0)
    Z = torch.full((batch, S * width), -3.0, device="cuda")
    _head_launch(_t(X), pq, ph, Z, S, D, batch, math=math, ld=ld, off=off)
    z = Z.cpu().numpy().reshape(batch, S, width)
    tol = TOL_TF32X3 if math == "tf32x3" else 5e-3
    for b in range(batch):
        assert normwise(z[b, :, off:off + dk].reshape(-1), ref[b]) <= tol, b
    if ld:
        mask = np.ones(width, bool)
        mask[off:off + dk] = False
        assert (z[:, :, mask] == -3.0).all()
