"""TMA-staged GEMMs next to a neighbour kernel that only HOLDS shared memory
(ttk_debug_occupy): which property of a co-resident kernel corrupts them
(DESIGN 6.2)?  python tools/overlap_tma_occupy.py smem_bytes threads mode"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2409_09471_b200 import _lib
lib = _lib.load(); dev = torch.device("cuda", 0)
smem = int(sys.argv[1]) if len(sys.argv) > 1 else 54784
thr = int(sys.argv[2]) if len(sys.argv) > 2 else 128
mode = int(sys.argv[3]) if len(sys.argv) > 3 else 0
shapes = [(80, 10240, 192), (80, 24576, 192), (24576, 80, 192)]
g = torch.Generator(device=dev); g.manual_seed(0)
sets = []
for r in range(6):
    M, N, K = shapes[r % 3]
    A = torch.randn((M, K), dtype=torch.float64, device=dev, generator=g)
    B = torch.randn((K, N), dtype=torch.float64, device=dev, generator=g)
    sets.append((M, N, K, A, B, torch.zeros((M, N), dtype=torch.float64, device=dev), A @ B))
src = torch.randn(4096, dtype=torch.float64, device=dev, generator=g)
bad = torch.zeros(1, dtype=torch.int32, device=dev)
S1, S2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
torch.cuda.synchronize()
wrong = 0
for rep in range(40):
    for r in range(6):
        _lib.check(lib.ttk_debug_occupy(148, thr, smem, 20000, mode, src.data_ptr(), bad.data_ptr(), S2.cuda_stream))
        M, N, K, A, B, C, ref = sets[r]
        _lib.check(lib.ttk_gemm_tma_strided(M, N, K, 1.0, A.data_ptr(), K, 1, B.data_ptr(), N, 1, 0.0, C.data_ptr(), N, 1,
                                            None, 0, S1.cuda_stream))
    torch.cuda.synchronize()
    for (M, N, K, A, B, C, ref) in sets:
        if float((C - ref).abs().max()) > 1e-8 * K: wrong += 1
        C.zero_()
    torch.cuda.synchronize()
print("neighbour smem", smem, "threads", thr, "mode", mode, ": wrong TMA outputs", wrong, "of", 240, "; neighbour words corrupted", int(bad.item()))
