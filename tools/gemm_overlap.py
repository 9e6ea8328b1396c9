"""TMA GEMMs of DIFFERENT problems overlapping on the GPU: one host thread,
several streams, many small launches without host syncs, rotating buffers so
every launch has its own tensor maps (diagnostics)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2409_09471_b200 import _lib
lib = _lib.load(); dev = torch.device("cuda", 0)
ns = int(sys.argv[1]) if len(sys.argv) > 1 else 3
shapes = [(80, 10240, 192), (80, 24576, 192), (24576, 80, 192), (80, 2048, 192), (2048, 80, 64)]
R = 8
S = [torch.cuda.Stream(dev) for _ in range(ns)]
data = []
for i in range(ns):
    g = torch.Generator(device=dev); g.manual_seed(i)
    sets = []
    for r in range(R):
        M, N, K = shapes[(i + r) % len(shapes)]
        A = torch.randn((M, K), dtype=torch.float64, device=dev, generator=g)
        B = torch.randn((K, N), dtype=torch.float64, device=dev, generator=g)
        sets.append((M, N, K, A, B, torch.zeros((M, N), dtype=torch.float64, device=dev), A @ B))
    data.append(sets)
torch.cuda.synchronize()
bad = 0
for rep in range(40):
    for r in range(R):
        for i, s in enumerate(S):
            M, N, K, A, B, C, ref = data[i][r]
            _lib.check(lib.ttk_gemm_tma_strided(M, N, K, 1.0, A.data_ptr(), K, 1, B.data_ptr(), N, 1, 0.0, C.data_ptr(), N, 1,
                                                None, 0, s.cuda_stream))
    torch.cuda.synchronize()
    for i in range(ns):
        for (M, N, K, A, B, C, ref) in data[i]:
            e = float((C - ref).abs().max())
            if e > 1e-9:
                bad += 1
            C.zero_()
    torch.cuda.synchronize()
print("streams", ns, "wrong outputs", bad, "of", 40 * R * ns)
