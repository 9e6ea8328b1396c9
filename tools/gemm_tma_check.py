"""ttk_gemm_tma_strided against torch on every operand layout (row-major /
transposed A and B, row- / column-major C), split-K shapes, padded leading
dimensions; timing beside the grouped cp.async kernel (diagnostics)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2409_09471_b200 import _lib
lib = _lib.load(); dev = torch.device("cuda", 0); st = _lib.stream_ptr(dev)
g = torch.Generator(device=dev).manual_seed(0)
ws = torch.empty(64 << 20, dtype=torch.uint8, device=dev)


def timed(f, reps=20):
    for _ in range(3): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


def case(M, N, K, ta, tb, tc, pad=0):
    A0 = torch.randn((K, M + pad) if ta else (M, K + pad), dtype=torch.float64, device=dev, generator=g)
    B0 = torch.randn((N, K + pad) if tb else (K, N + pad), dtype=torch.float64, device=dev, generator=g)
    A = A0[:, :M].t() if ta else A0[:, :K]
    B = B0[:, :K].t() if tb else B0[:, :N]
    ref = A @ B
    C0 = torch.full((N, M + pad) if tc else (M, N + pad), 3.0, dtype=torch.float64, device=dev)
    a_ms, a_ks = (1, M + pad) if ta else (K + pad, 1)
    b_ks, b_ns = (1, K + pad) if tb else (N + pad, 1)
    c_ms, c_ns = (1, M + pad) if tc else (N + pad, 1)
    f = lambda: lib.ttk_gemm_tma_strided(M, N, K, 1.0, A0.data_ptr(), a_ms, a_ks, B0.data_ptr(), b_ks, b_ns, 0.0,
                                         C0.data_ptr(), c_ms, c_ns, ws.data_ptr(), ws.numel(), st)
    _lib.check(f())
    torch.cuda.synchronize()
    C = C0[:, :M].t() if tc else C0[:, :N]
    err = (C - ref).abs().max().item() / ref.abs().max().item()
    t = timed(f)
    h = lambda: lib.ttk_gemm_strided(1, M, N, K, 1.0, A0.data_ptr(), a_ms, a_ks, 0, B0.data_ptr(), b_ks, b_ns, 0, 0.0,
                                     C0.data_ptr(), c_ms, c_ns, 0, ws.data_ptr(), ws.numel(), st)
    t0 = timed(h)
    print(f"{M}x{N}x{K} TA={int(ta)} TB={int(tb)} colC={int(tc)} pad={pad}: err {err:.1e}  tma {t:6.1f} us  "
          f"grouped {t0:6.1f} us", flush=True)


for args in [(192, 80, 10240, False, True, False), (80, 192, 10240, True, False, False),
             (80, 80, 8192, False, True, False), (8192, 64, 80, True, False, True), (24576, 80, 192, False, False, False),
             (80, 24576, 192, False, False, False), (100, 130, 50, True, True, False, 2), (96, 40, 300, True, True, True, 4),
             (64, 64, 1000, False, False, True, 2)]:
    case(*args)
