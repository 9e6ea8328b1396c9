"""Cluster Jacobi with vs without V accumulation (upper bound for offloading V)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2409_09471_b200 import _lib
lib = _lib.load(); dev = torch.device("cuda", 0); st = _lib.stream_ptr(dev)
res = {}
for l in (40, 80, 128):
    g = torch.Generator().manual_seed(0)
    R = torch.linalg.qr(torch.randn(10 * l, l, dtype=torch.float64, generator=g))[1].T.contiguous().to(dev)
    U = torch.empty((l, l), dtype=torch.float64, device=dev); S = torch.empty(l, dtype=torch.float64, device=dev)
    V = torch.empty((l, l), dtype=torch.float64, device=dev)
    for name, vp in (("with_v", V.data_ptr()), ("no_v", None)):
        f = lambda: lib.ttk_svd_small(l, l, R.data_ptr(), U.data_ptr(), S.data_ptr(), vp, st)
        f(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); [f() for _ in range(10)]; b.record(); torch.cuda.synchronize()
        res[f"{l}_{name}"] = round(a.elapsed_time(b) / 10 * 1e3, 1)
print(json.dumps(res))
