"""Host cost of one hs_launch call (GEMM, GEMM_NT, add) and of an event create/record/wait/
destroy cycle, from Python through ctypes: the per-command cost behind dynamic-mode dispatch."""
import ctypes, sys, time
sys.path.insert(0, ".")
import torch
from paper_2009_07482_b200 import _native
from tests.gpu_util import stream
L = _native.lib(); st = stream()
def mk(op, M, N, K):
    A = torch.randn(M*K, device="cuda"); B = torch.randn(N*K, device="cuda"); C = torch.empty(M*N, device="cuda")
    a = _native.OpArgs(); a.n_in = 2; a.in_[0], a.in_[1] = A.data_ptr(), B.data_ptr(); a.in_stride[0]=M*K; a.in_stride[1]=N*K
    a.out, a.out_stride = C.data_ptr(), M*N; a.dims[0], a.dims[1], a.dims[2] = M, N, K
    return (A,B,C,a)
for name, op, dims in (("gemm", 0, (128,64,512)), ("gemm_nt", 1, (128,128,64)), ("add", 6, (65536,0,0))):
    keep = mk(op, *dims) if op != 6 else None
    if op == 6:
        A = torch.randn(65536, device="cuda"); B = torch.randn(65536, device="cuda"); C = torch.empty(65536, device="cuda")
        a = _native.OpArgs(); a.n_in=2; a.in_[0], a.in_[1] = A.data_ptr(), B.data_ptr(); a.in_stride[0]=a.in_stride[1]=65536
        a.out, a.out_stride = C.data_ptr(), 65536; a.dims[0]=65536; keep=(A,B,C,a)
    a = keep[3]
    torch.cuda.synchronize()
    for _ in range(10): _native.check(L.hs_launch(st, op, ctypes.byref(a), 0, 1))
    _native.check(L.hs_stream_sync(st))
    t0 = time.perf_counter(); n = 500
    for _ in range(n): L.hs_launch(st, op, ctypes.byref(a), 0, 1)
    t1 = time.perf_counter()
    _native.check(L.hs_stream_sync(st))
    print(f"{name}: host {1e6*(t1-t0)/n:.1f} us per hs_launch")
ev = ctypes.c_void_p(); ctx = ctypes.c_void_p(); _native.check(L.hs_ctx_create(0, ctypes.byref(ctx)))
t0 = time.perf_counter()
for _ in range(200):
    _native.check(L.hs_event_create(ctx, 0, ctypes.byref(ev))); L.hs_event_record(ev, st); L.hs_stream_wait(st, ev); L.hs_event_destroy(ev)
print(f"event create+record+wait+destroy: {1e6*(time.perf_counter()-t0)/200:.1f} us")
