"""One CholeskyQR2 (10240 x 80 Gaussian) for ncu: blocked Cholesky, near-identity series, TRSM, GEMMs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2409_09471_b200 import _lib
lib = _lib.load(); dev = torch.device("cuda", 0); st = _lib.stream_ptr(dev)
m, l = 10240, 80
A = torch.as_tensor(np.random.default_rng(0).standard_normal((m, l)), device=dev)
Q = torch.empty_like(A); R = torch.empty((l, l), dtype=torch.float64, device=dev)
ws = _lib.workspace(lib.ttk_qr_ws_bytes(m, l) + (64 << 20), dev)
for _ in range(3):
    assert lib.ttk_qr_auto(m, l, A.data_ptr(), l, 1, Q.data_ptr(), l, 1, R.data_ptr(), ws.data_ptr(), ws.numel(), st) == 0
torch.cuda.synchronize(); print("ok")
if len(sys.argv) > 1 and sys.argv[1] == "prof":
    ts = torch.zeros(16, dtype=torch.int64, device=dev)
    lib.ttk_debug_fused_qr_profile(ts.data_ptr())
    lib.ttk_qr_auto(m, l, A.data_ptr(), l, 1, Q.data_ptr(), l, 1, R.data_ptr(), ws.data_ptr(), ws.numel(), st)
    torch.cuda.synchronize(); lib.ttk_debug_fused_qr_profile(None)
    t = ts.cpu().numpy(); names = ["load+gram1", "reduce1", "chol1", "trsm+gram2", "reduce2", "nearid+R", "Q"]
    idx = [0, 1, 2, 3, 4, 5, 6, 15]
    print({names[i]: round((t[idx[i + 1]] - t[idx[i]]) / 1e3, 2) for i in range(7)}, "total_us", (t[15] - t[0]) / 1e3)
