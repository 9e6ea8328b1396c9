"""The suspected pairing of DESIGN 6.2 in isolation: TMA-staged GEMMs on some
streams next to grouped cp.async GEMMs (ttk_gemm_strided, incl. the long-K
split-K shapes of the sweeps) on others, static inputs, one host thread, no host
syncs inside a round; every output of both kinds is checked (diagnostics)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2409_09471_b200 import _lib
lib = _lib.load(); dev = torch.device("cuda", 0)
tma_shapes = [(80, 10240, 192), (80, 24576, 192), (24576, 80, 192)]
grp_shapes = [(192, 80, 10240), (80, 192, 10240), (24576, 384, 128)]
nst = int(sys.argv[1]) if len(sys.argv) > 1 else 2
if len(sys.argv) > 2:  # restrict the grouped neighbour to one shape: M,N,K
    grp_shapes = [tuple(int(v) for v in sys.argv[2].split(","))]
if len(sys.argv) > 3:
    tma_shapes = [tuple(int(v) for v in sys.argv[3].split(","))]
g = torch.Generator(device=dev); g.manual_seed(0)
def mk(shapes, reps):
    sets = []
    for r in range(reps):
        M, N, K = shapes[r % len(shapes)]
        A = torch.randn((M, K), dtype=torch.float64, device=dev, generator=g)
        B = torch.randn((K, N), dtype=torch.float64, device=dev, generator=g)
        sets.append((M, N, K, A, B, torch.zeros((M, N), dtype=torch.float64, device=dev), A @ B))
    return sets
ST = [torch.cuda.Stream(dev) for _ in range(nst)]; SG = [torch.cuda.Stream(dev) for _ in range(nst)]
tma = [mk(tma_shapes, 6) for _ in range(nst)]; grp = [mk(grp_shapes, 6) for _ in range(nst)]
wsb = max(lib.ttk_gemm_strided_ws_bytes(1, M, N, K) for (M, N, K) in grp_shapes) + (32 << 20)
wss = [torch.empty(wsb, dtype=torch.uint8, device=dev) for _ in range(nst)]
TRANS = os.environ.get("TRANS") == "1"
tmaT = [[(A.t().contiguous(), B.t().contiguous()) for (M, N, K, A, B, C, ref) in sets] for sets in tma]
torch.cuda.synchronize()
bad_t = bad_g = 0
for rep in range(60):
    for r in range(6):
        for i in range(nst):
            M, N, K, A, B, C, ref = tma[i][r]
            if TRANS:  # A^T, B^T stored row-major and a column-major C: the TA / TB instances
                At, Bt = tmaT[i][r]
                _lib.check(lib.ttk_gemm_tma_strided(M, N, K, 1.0, At.data_ptr(), 1, M, Bt.data_ptr(), 1, K, 0.0, C.data_ptr(),
                                                    N, 1, None, 0, ST[i].cuda_stream))
            else:
                _lib.check(lib.ttk_gemm_tma_strided(M, N, K, 1.0, A.data_ptr(), K, 1, B.data_ptr(), N, 1, 0.0, C.data_ptr(), N, 1,
                                                    None, 0, ST[i].cuda_stream))
            M, N, K, A, B, C, ref = grp[i][r]
            if os.environ.get("NEIGHBOUR") == "cublas":
                with torch.cuda.stream(SG[i]):
                    torch.matmul(A, B, out=C)
                continue
            _lib.check(lib.ttk_gemm_strided(1, M, N, K, 1.0, A.data_ptr(), K, 1, 0, B.data_ptr(), N, 1, 0, 0.0, C.data_ptr(), N, 1, 0,
                                            wss[i].data_ptr(), wss[i].numel(), SG[i].cuda_stream))
    torch.cuda.synchronize()
    for i in range(nst):
        for (M, N, K, A, B, C, ref) in tma[i]:
            if float((C - ref).abs().max()) > 1e-8 * K: bad_t += 1
            C.zero_()
        for (M, N, K, A, B, C, ref) in grp[i]:
            if float((C - ref).abs().max()) > 1e-8 * K: bad_g += 1
            C.zero_()
    torch.cuda.synchronize()
print("stream pairs", nst, ": wrong TMA outputs", bad_t, ", wrong grouped outputs", bad_g, "of", 60 * 6 * nst, "each")
