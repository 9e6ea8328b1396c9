"""ttk_gemm_tma against torch on shapes that hit every tile variant, with
padded leading dimensions and offset bases (diagnostics)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2409_09471_b200 import _lib
lib = _lib.load(); dev = torch.device("cuda", 0); st = _lib.stream_ptr(dev)
g = torch.Generator(device=dev).manual_seed(0)
for (M, N, K, pa, pb, pc) in [(24576, 80, 192, 0, 0, 0), (80, 24576, 192, 0, 0, 0), (80, 10240, 192, 0, 0, 0),
                             (10240, 64, 80, 0, 16, 0), (10240, 64, 80, 0, 0, 0), (8192, 64, 80, 0, 0, 0),
                             (80, 4096, 100, 0, 0, 0), (1000, 80, 40, 4, 2, 6), (100, 130, 50, 2, 6, 4)]:
    A = torch.randn(M, K + pa, dtype=torch.float64, device=dev, generator=g)
    B = torch.randn(K, N + pb, dtype=torch.float64, device=dev, generator=g)
    C = torch.full((M, N + pc), 7.0, dtype=torch.float64, device=dev)
    ref = A[:, :K] @ B[:, :N]
    _lib.check(lib.ttk_gemm_tma(M, N, K, 1.0, A.data_ptr(), K + pa, B.data_ptr(), N + pb, 0.0, C.data_ptr(), N + pc, st))
    torch.cuda.synchronize()
    err = (C[:, :N] - ref).abs().max().item() / (ref.abs().max().item())
    pad_ok = bool((C[:, N:] == 7.0).all().item()) if pc else True
    print(f"{M}x{N}x{K} pads {pa},{pb},{pc}: rel err {err:.1e} pad untouched {pad_ok}", flush=True)
