"""Jacobi SVD of exactly low-rank (cross-matrix-like) inputs vs LAPACK: the small singular values."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2409_09471_b200 import _lib
lib = _lib.load()
dev = torch.device("cuda", 0)


def svd_gpu(B):
    k, l = B.shape
    kn = min(k, l)
    Bt = torch.as_tensor(B, device=dev)
    U = torch.empty((k, kn), dtype=torch.float64, device=dev)
    S = torch.empty(kn, dtype=torch.float64, device=dev)
    V = torch.empty((l, kn), dtype=torch.float64, device=dev)
    _lib.check(lib.ttk_svd_small(k, l, Bt.data_ptr(), U.data_ptr(), S.data_ptr(), V.data_ptr(), _lib.stream_ptr(dev)))
    return S.cpu().numpy(), U.cpu().numpy(), V.cpu().numpy()


rng = np.random.default_rng(0)
for (k, l, r) in [(60, 40, 5), (60, 40, 1), (40, 40, 5), (80, 60, 7), (120, 100, 10), (30, 20, 3)]:
    B = rng.standard_normal((k, r)) @ rng.standard_normal((r, l))
    s, u, v = svd_gpu(B)
    sl = np.linalg.svd(B, compute_uv=False)
    print(f"{k}x{l} rank {r}: kept(1e-12) gpu {np.sum(s > 1e-12 * s[0])} lapack {np.sum(sl > 1e-12 * sl[0])}; "
          f"gpu s[r]/s0 {s[r] / s[0]:.2e} lapack {sl[r] / sl[0]:.2e}; rec {np.linalg.norm((u * s) @ v.T - B) / np.linalg.norm(B):.1e}")
