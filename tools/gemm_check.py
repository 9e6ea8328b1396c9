"""Correctness sweep of ttk_gemm_strided over forced tile configs and layouts (diagnostics)."""
import os, sys, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2409_09471_b200 import _lib
lib = _lib.load(); dev = torch.device("cuda", 0); st = _lib.stream_ptr(dev)
def run(M, N, K, layout):
    g = torch.Generator().manual_seed(1)
    A = torch.randn(M * K, dtype=torch.float64, generator=g); B = torch.randn(K * N, dtype=torch.float64, generator=g)
    if layout == "nn": (ams, aks), (bks, bns) = (K, 1), (N, 1)
    elif layout == "tn": (ams, aks), (bks, bns) = (1, M), (N, 1)
    else: (ams, aks), (bks, bns) = (K, 1), (1, K)
    ref = torch.as_strided(A, (M, K), (ams, aks)) @ torch.as_strided(B, (K, N), (bks, bns))
    dA, dB = A.to(dev), B.to(dev); C = torch.zeros(M, N, dtype=torch.float64, device=dev)
    ws = _lib.workspace(int(lib.ttk_gemm_strided_ws_bytes(1, M, N, K)) + 8, dev)
    rc = lib.ttk_gemm_strided(1, M, N, K, 1.0, dA.data_ptr(), ams, aks, 0, dB.data_ptr(), bks, bns, 0, 0.0, C.data_ptr(), N, 1, 0, ws.data_ptr(), ws.numel(), st)
    torch.cuda.synchronize()
    return rc, (C.cpu() - ref).abs().max().item() / ref.abs().max().item()
cfg = os.environ.get("TTK_GEMM_FORCE_CFG", "auto")
for M, N, K in [(80, 192, 1024), (80, 192, 64), (160, 128, 64), (80, 64, 16), (96, 64, 32)]:
    for layout in ("nn", "tn", "nt"):
        rc, e = run(M, N, K, layout)
        print(f"cfg={cfg} {M}x{N}x{K} {layout} rc={rc} rel={e:.1e}{'  <-- BAD' if e > 1e-12 else ''}")
