"""Host cost per ABI call (ctypes + C++ planning + CUDA launch) for a trivial
elementwise kernel and for a tiny GEMM (diagnostics)."""
import os, sys, time, json, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2409_09471_b200 import _lib
lib = _lib.load(); dev = torch.device("cuda", 0); st = _lib.stream_ptr(dev)
x = torch.ones(64, dtype=torch.float64, device=dev)
A = torch.randn(64, 16, dtype=torch.float64, device=dev); B = torch.randn(16, 16, dtype=torch.float64, device=dev)
C = torch.empty(64, 16, dtype=torch.float64, device=dev)
ws = _lib.workspace(1 << 20, dev)
res = {}
def loop(name, fn, n=20000):
    for _ in range(100): fn()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n): fn()
    t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    res[name] = {"host_us_per_call": (t1 - t0) / n * 1e6, "wall_us_per_call": (t2 - t0) / n * 1e6}
loop("scale", lambda: lib.ttk_scale(x.data_ptr(), x.data_ptr(), 64, 1.0, st))
loop("gemm_64x16x16", lambda: lib.ttk_gemm_strided(1, 64, 16, 16, 1.0, A.data_ptr(), 16, 1, 0, B.data_ptr(), 16, 1, 0, 0.0, C.data_ptr(), 16, 1, 0, ws.data_ptr(), ws.numel(), st))
loop("torch_add", lambda: x.add_(0.0))
print(json.dumps(res, indent=1))
