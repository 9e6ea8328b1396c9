"""TF/s of every forced tile config on the workload's GEMM shapes (run once per
config via TTK_GEMM_FORCE_CFG; prints one JSON line)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2409_09471_b200 import _lib
lib = _lib.load(); dev = torch.device("cuda", 0); st = _lib.stream_ptr(dev)
def t_ev(fn, reps=20):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); [fn() for _ in range(reps)]; b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e-3
res = {}
for (M, N, K) in [(24576, 80, 192), (80, 24576, 192), (10240, 80, 192), (80, 80, 10240), (80, 192, 10240), (192, 80, 10240),
                  (10240, 80, 80), (10240, 64, 80), (8192, 80, 80), (64, 8192, 80), (4096, 4096, 4096)]:
    A = torch.randn(M, K, dtype=torch.float64, device=dev); B = torch.randn(K, N, dtype=torch.float64, device=dev)
    C = torch.empty(M, N, dtype=torch.float64, device=dev)
    ws = _lib.workspace(int(lib.ttk_gemm_strided_ws_bytes(1, M, N, K)) + 8, dev)
    f = lambda: lib.ttk_gemm_strided(1, M, N, K, 1.0, A.data_ptr(), K, 1, 0, B.data_ptr(), N, 1, 0, 0.0, C.data_ptr(), N, 1, 0, ws.data_ptr(), ws.numel(), st)
    res[f"{M}x{N}x{K}"] = round(t_ev(f) * 1e6, 1)
print(json.dumps({"cfg": os.environ.get("TTK_GEMM_FORCE_CFG", "auto"), "us": res}))
