"""Time + check the truncation's SVD (ttk_svd_small, V accumulated) on l x l R^T factors."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2409_09471_b200 import _lib
lib = _lib.load()
dev = torch.device("cuda", 0)
st = torch.cuda.current_stream(dev)
for l in [int(a) for a in (sys.argv[1:] or ["80", "64", "48", "50", "96"])]:
    g = np.random.default_rng(l)
    R = np.linalg.qr(g.standard_normal((10 * l, l)))[1]
    B = np.ascontiguousarray(R.T)
    Bt = torch.as_tensor(B, device=dev)
    U = torch.empty((l, l), dtype=torch.float64, device=dev)
    S = torch.empty(l, dtype=torch.float64, device=dev)
    V = torch.empty((l, l), dtype=torch.float64, device=dev)
    call = lambda: lib.ttk_svd_small(l, l, Bt.data_ptr(), U.data_ptr(), S.data_ptr(), V.data_ptr(), st.cuda_stream)
    c1 = torch.zeros(1, dtype=torch.int32, device=dev)
    lib.ttk_debug_svd_sweeps(c1.data_ptr())
    _lib.check(call()); torch.cuda.synchronize()
    print("sweeps", int(c1.item()))
    lib.ttk_debug_svd_sweeps(None)
    for _ in range(3):
        _lib.check(call())
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(20):
        call()
    b.record(st)
    torch.cuda.synchronize()
    u, s, v = U.cpu().numpy(), S.cpu().numpy(), V.cpu().numpy()
    sl = np.linalg.svd(B, compute_uv=False)
    print(f"{l}x{l}: {a.elapsed_time(b) / 20 * 1e3:.1f} us; |S-S_lapack|/S0 {np.abs(s - sl).max() / sl[0]:.1e} "
          f"U orth {np.abs(u.T @ u - np.eye(l)).max():.1e} V orth {np.abs(v.T @ v - np.eye(l)).max():.1e} "
          f"res {np.linalg.norm(B @ v - u * s) / np.linalg.norm(B):.1e}", flush=True)
