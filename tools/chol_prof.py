"""Phase clocks of the blocked Cholesky inside one CholeskyQR2 (diagnostics)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2409_09471_b200 import _lib
lib = _lib.load(); dev = torch.device("cuda", 0); st = _lib.stream_ptr(dev)
m, l = 10240, 80
A = torch.as_tensor(np.random.default_rng(0).standard_normal((m, l)), device=dev)
Q = torch.empty_like(A); R = torch.empty((l, l), dtype=torch.float64, device=dev)
ws = _lib.workspace(lib.ttk_qr_ws_bytes(m, l) + (64 << 20), dev)
lib.ttk_qr_auto(m, l, A.data_ptr(), l, 1, Q.data_ptr(), l, 1, R.data_ptr(), ws.data_ptr(), ws.numel(), st)
prof = torch.zeros(8, dtype=torch.int64, device=dev)
lib.ttk_debug_chol_profile(prof.data_ptr())
lib.ttk_qr_auto(m, l, A.data_ptr(), l, 1, Q.data_ptr(), l, 1, R.data_ptr(), ws.data_ptr(), ws.numel(), st)
torch.cuda.synchronize(); lib.ttk_debug_chol_profile(None)
p = prof.cpu().numpy()
n = max(p[5], 1)
print("calls", p[5], "cycles per call: load", p[0] / n, "diag", p[1] / n, "panel", p[2] / n, "trailing", p[3] / n, "epilogue", p[4] / n)
