"""qr_auto time per shape (CholeskyQR2 vs Householder via TTK_QR_MODE) -- diagnostics."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2409_09471_b200 import _lib
lib = _lib.load(); dev = torch.device("cuda", 0); st = _lib.stream_ptr(dev)
res = {"mode": os.environ.get("TTK_QR_MODE", "0")}
for m, l in [(128, 80), (256, 40), (32, 20), (512, 100), (1000, 80), (256, 20), (640, 60), (10240, 80)]:
    A = torch.as_tensor(np.random.default_rng(0).standard_normal((m, l)), device=dev)
    Q = torch.empty_like(A); R = torch.empty((l, l), dtype=torch.float64, device=dev)
    ws = _lib.workspace(lib.ttk_qr_ws_bytes(m, l) + (64 << 20), dev)
    f = lambda: lib.ttk_qr_auto(m, l, A.data_ptr(), l, 1, Q.data_ptr(), l, 1, R.data_ptr(), ws.data_ptr(), ws.numel(), st)
    for _ in range(3): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10): f()
    b.record(); torch.cuda.synchronize()
    q, r = Q.cpu().numpy(), R.cpu().numpy()
    res[f"{m}x{l}"] = (round(a.elapsed_time(b) / 10 * 1e3, 1), float(np.abs(q.T @ q - np.eye(l)).max()),
                       float(np.abs(q @ r - A.cpu().numpy()).max()))
print(json.dumps(res))
