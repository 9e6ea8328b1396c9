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
