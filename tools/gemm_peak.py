"""TF/s of ttk_gemm_strided on plain square and skinny shapes vs torch (cuBLAS) fp64."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2409_09471_b200 import _lib
lib = _lib.load(); dev = torch.device("cuda", 0); st = _lib.stream_ptr(dev)
def t_ev(fn, reps=10):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); [fn() for _ in range(reps)]; b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e-3
res = {}
shapes = [(4096, 4096, 4096), (8192, 8192, 2048), (24576, 80, 192), (10240, 80, 80), (80, 80, 10240), (4096, 384, 128)]
if len(sys.argv) > 1:
    shapes = [tuple(int(x) for x in a.split("x")) for a in sys.argv[1:]]
for (M, N, K) in shapes:
    A = torch.randn(M, K, dtype=torch.float64, device=dev); B = torch.randn(K, N, dtype=torch.float64, device=dev)
    C = torch.empty(M, N, dtype=torch.float64, device=dev)
    ws = _lib.workspace(int(lib.ttk_gemm_strided_ws_bytes(1, M, N, K)) + 8, dev)
    f = lambda: lib.ttk_gemm_strided(1, M, N, K, 1.0, A.data_ptr(), K, 1, 0, B.data_ptr(), N, 1, 0, 0.0, C.data_ptr(), N, 1, 0, ws.data_ptr(), ws.numel(), st)
    t = t_ev(f); tc = t_ev(lambda: torch.mm(A, B, out=C))
    res[f"{M}x{N}x{K}"] = {"ttk_tfs": round(2 * M * N * K / t / 1e12, 2), "cublas_tfs": round(2 * M * N * K / tc / 1e12, 2), "ttk_us": round(t * 1e6, 1), "cublas_us": round(tc * 1e6, 1)}
print(json.dumps(res, indent=1))
