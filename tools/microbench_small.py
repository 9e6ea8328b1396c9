"""Time the single-CTA kernels (Jacobi SVD, CholeskyQR2 via qr, TSQR) at solver/config sizes."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2409_09471_b200 import _lib
lib = _lib.load()
dev = torch.device("cuda", 0)
st = _lib.stream_ptr(dev)
res = {}
def ev_time(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); [fn() for _ in range(reps)]; b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3  # us
cnt = torch.zeros(1, dtype=torch.int32, device=dev)
lib.ttk_debug_svd_sweeps(cnt.data_ptr())
rng = np.random.default_rng(0)
for k in (20, 50, 80, 100, 120):
    B = torch.as_tensor(np.linalg.qr(rng.standard_normal((10 * k, k)))[1], device=dev)  # an R factor
    U = torch.empty((k, k), dtype=torch.float64, device=dev); S = torch.empty(k, dtype=torch.float64, device=dev)
    us = ev_time(lambda: lib.ttk_svd_small(k, k, B.data_ptr(), U.data_ptr(), S.data_ptr(), None, st))
    res[f"svd_{k}"] = {"us": us, "sweeps": int(cnt.item())}
lib.ttk_debug_svd_sweeps(None)
for m, l in ((10240, 80), (3200, 50), (25600, 100), (8192, 64)):
    A = torch.as_tensor(rng.standard_normal((m, l)), device=dev)
    Q = torch.empty((m, l), dtype=torch.float64, device=dev); R = torch.empty((l, l), dtype=torch.float64, device=dev)
    ws = _lib.workspace(lib.ttk_qr_ws_bytes(m, l) + (64 << 20), dev)
    us = ev_time(lambda: lib.ttk_qr(m, l, A.data_ptr(), l, 1, Q.data_ptr(), l, 1, R.data_ptr(), ws.data_ptr(), ws.numel(), st))
    res[f"qr_{m}x{l}"] = {"us": us}
print(json.dumps(res, indent=1))
