"""Concurrency check of the TMA GEMM from ONE host thread: launches alternate
between two streams with separate buffers (diagnostics)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2409_09471_b200 import _lib
lib = _lib.load(); dev = torch.device("cuda", 0)
shapes = [(24576, 80, 192), (80, 24576, 192), (80, 10240, 192), (8192, 64, 80), (80, 80, 8192)]
S = [torch.cuda.Stream(dev) for _ in range(2)]
data = []
for i, s in enumerate(S):
    with torch.cuda.stream(s):
        g = torch.Generator(device=dev); g.manual_seed(i)
        ws = torch.empty(32 << 20, dtype=torch.uint8, device=dev)
        sets = []
        for (M, N, K) in shapes:
            A = torch.randn((M, K), dtype=torch.float64, device=dev, generator=g)
            B = torch.randn((K, N), dtype=torch.float64, device=dev, generator=g)
            sets.append((M, N, K, A, B, torch.empty((M, N), dtype=torch.float64, device=dev), A @ B))
        data.append((ws, sets))
torch.cuda.synchronize()
worst = [0.0, 0.0]
for rep in range(20):
    for j in range(len(shapes)):
        for i, s in enumerate(S):
            ws, sets = data[i]
            M, N, K, A, B, C, ref = sets[j]
            _lib.check(lib.ttk_gemm_tma_strided(M, N, K, 1.0, A.data_ptr(), K, 1, B.data_ptr(), N, 1, 0.0, C.data_ptr(), N, 1,
                                                ws.data_ptr(), ws.numel(), s.cuda_stream))
    torch.cuda.synchronize()
    for i in range(2):
        for (M, N, K, A, B, C, ref) in data[i][1]:
            worst[i] = max(worst[i], float((C - ref).abs().max()))
print("max |C - AB| per stream", worst)
