"""TMA GEMMs on some streams overlapping fused CholeskyQR2 launches on others
(one host thread, no syncs inside a round); every output is checked (diagnostics)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2409_09471_b200 import _lib
lib = _lib.load(); dev = torch.device("cuda", 0)
shapes = [(80, 10240, 192), (80, 24576, 192), (24576, 80, 192)]
m, l = 10240, 80
SG = [torch.cuda.Stream(dev) for _ in range(2)]
SQ = [torch.cuda.Stream(dev) for _ in range(2)]
g = torch.Generator(device=dev); g.manual_seed(0)
gem = []
for i in range(2):
    sets = []
    for r in range(6):
        M, N, K = shapes[(i + r) % 3]
        A = torch.randn((M, K), dtype=torch.float64, device=dev, generator=g)
        B = torch.randn((K, N), dtype=torch.float64, device=dev, generator=g)
        sets.append((M, N, K, A, B, torch.zeros((M, N), dtype=torch.float64, device=dev), A @ B))
    gem.append(sets)
qrs = []
for i in range(2):
    A = torch.randn((m, l), dtype=torch.float64, device=dev, generator=g)
    qrs.append((A, torch.zeros_like(A), torch.zeros((l, l), dtype=torch.float64, device=dev),
                torch.empty(lib.ttk_qr_ws_bytes(m, l) + (64 << 20), dtype=torch.uint8, device=dev)))
torch.cuda.synchronize()
bad_g = bad_q = 0
eye = torch.eye(l, device=dev, dtype=torch.float64)
for rep in range(60):
    for r in range(6):
        for i in range(2):
            M, N, K, A, B, C, ref = gem[i][r]
            _lib.check(lib.ttk_gemm_tma_strided(M, N, K, 1.0, A.data_ptr(), K, 1, B.data_ptr(), N, 1, 0.0, C.data_ptr(), N, 1,
                                                None, 0, SG[i].cuda_stream))
            A2, Q, R, ws = qrs[i]
            _lib.check(lib.ttk_qr_auto(m, l, A2.data_ptr(), l, 1, Q.data_ptr(), l, 1, R.data_ptr(), ws.data_ptr(), ws.numel(),
                                       SQ[i].cuda_stream))
    torch.cuda.synchronize()
    for i in range(2):
        for (M, N, K, A, B, C, ref) in gem[i]:
            if float((C - ref).abs().max()) > 1e-9: bad_g += 1
            C.zero_()
        A2, Q, R, ws = qrs[i]
        if float((Q @ R - A2).abs().max()) > 1e-9 or float((Q.T @ Q - eye).abs().max()) > 1e-9: bad_q += 1
        Q.zero_(); R.zero_()
    torch.cuda.synchronize()
print("wrong gemm outputs", bad_g, "of", 60 * 12, "; wrong QRs", bad_q, "of", 120)
