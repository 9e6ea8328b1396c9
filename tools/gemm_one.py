"""One 4096^3 fp64 GEMM through ttk_gemm_strided (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2409_09471_b200 import _lib
lib = _lib.load(); dev = torch.device("cuda", 0); st = _lib.stream_ptr(dev)
M = N = K = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
A = torch.randn(M, K, dtype=torch.float64, device=dev); B = torch.randn(K, N, dtype=torch.float64, device=dev)
C = torch.empty(M, N, dtype=torch.float64, device=dev)
ws = _lib.workspace(int(lib.ttk_gemm_strided_ws_bytes(1, M, N, K)) + 8, dev)
for _ in range(2):
    lib.ttk_gemm_strided(1, M, N, K, 1.0, A.data_ptr(), K, 1, 0, B.data_ptr(), N, 1, 0, 0.0, C.data_ptr(), N, 1, 0, ws.data_ptr(), ws.numel(), st)
torch.cuda.synchronize(); print("ok")
