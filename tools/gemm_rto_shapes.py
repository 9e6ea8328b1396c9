"""Time the config-3 RTO / truncation GEMM shapes through ttk_gemm_strided beside
cuBLAS (torch.mm, fp64), row-major operands; TF/s per shape (diagnostics)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2409_09471_b200 import _lib
lib = _lib.load(); dev = torch.device("cuda", 0); st = _lib.stream_ptr(dev)
SHAPES = [(24576, 80, 192), (80, 24576, 192), (80, 10240, 192), (192, 80, 10240), (80, 192, 10240),
          (10240, 64, 80), (8192, 64, 80), (80, 80, 8192)]
if len(sys.argv) > 1:
    SHAPES = [tuple(int(v) for v in a.split("x")) for a in sys.argv[1:]]


def timed(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


for M, N, K in SHAPES:
    A = torch.randn(M, K, dtype=torch.float64, device=dev)
    B = torch.randn(K, N, dtype=torch.float64, device=dev)
    C = torch.empty(M, N, dtype=torch.float64, device=dev)
    ws = _lib.workspace(int(lib.ttk_gemm_strided_ws_bytes(1, M, N, K)) + 8, dev)
    f = lambda: lib.ttk_gemm_strided(1, M, N, K, 1.0, A.data_ptr(), K, 1, 0, B.data_ptr(), N, 1, 0, 0.0,
                                     C.data_ptr(), N, 1, 0, ws.data_ptr(), ws.numel(), st)
    t = timed(f)
    ref = A @ B
    err = (C - ref).abs().max().item() / (A.abs().max().item() * B.abs().max().item() * K)
    C.zero_()
    g = lambda: lib.ttk_gemm_tma(M, N, K, 1.0, A.data_ptr(), K, B.data_ptr(), N, 0.0, C.data_ptr(), N, st)
    _lib.check(g())
    tt = timed(g)
    err_t = (C - ref).abs().max().item() / (A.abs().max().item() * B.abs().max().item() * K)
    tc = timed(lambda: torch.mm(A, B, out=C))
    fl = 2.0 * M * N * K
    print(f"M={M:6d} N={N:6d} K={K:6d}: ttk {t:7.1f} us {fl / t / 1e6:6.2f} TF/s | tma {tt:7.1f} us "
          f"{fl / tt / 1e6:6.2f} TF/s | cuBLAS {tc:7.1f} us {fl / tc / 1e6:6.2f} TF/s | err {err:.1e} tma {err_t:.1e}",
          flush=True)
