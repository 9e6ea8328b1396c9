"""Time + check the truncation's Gram eigensolver (ttk_gram_eig) against numpy
eigh, beside the QR + one-sided Jacobi SVD it replaces (ttk_svd_small on R^T).

usage: python tools/eig_one.py [n ...]   (default 80 64 50 128 33)
Inputs: C = Q diag(sigma) W^T (n x 10n) with the config-3-like spectrum
sigma_i = 1 - 0.3 i/n for the top 80 %, 0.12 - 0.02 i/n for the rest.
"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2409_09471_b200 import _lib
print("start", flush=True)
lib = _lib.load()
TRACE = torch.zeros(16, dtype=torch.int32).pin_memory()
lib.ttk_debug_gram_eig(int(os.environ.get('EIG_DBG', '0')), TRACE.data_ptr() if os.environ.get('EIG_TRACE') else None)
dev = torch.device("cuda", 0)
st = torch.cuda.current_stream(dev)


def timed(call, reps=20):
    for _ in range(3):
        _lib.check(call())
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps):
        call()
    b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


for n in [int(a) for a in (sys.argv[1:] or ["80", "64", "50", "128", "33"])]:
    g = np.random.default_rng(n)
    keep = int(0.8 * n)
    sig = np.concatenate([1 - 0.3 * np.arange(keep) / n, 0.12 - 0.02 * np.arange(n - keep) / n])
    q = np.linalg.qr(g.standard_normal((n, n)))[0]
    w = np.linalg.qr(g.standard_normal((10 * n, n)))[0]
    C = (q * sig) @ w.T
    G = C @ C.T
    Gt = torch.as_tensor(G, device=dev)
    S = torch.empty(n, dtype=torch.float64, device=dev)
    T1 = torch.zeros((n, n), dtype=torch.float64, device=dev)
    L = torch.zeros((n, n), dtype=torch.float64, device=dev)
    U = torch.empty((n, n), dtype=torch.float64, device=dev)
    info = torch.zeros(16, dtype=torch.int32, device=dev)
    call = lambda: lib.ttk_gram_eig(n, Gt.data_ptr(), n, 0.0, keep, S.data_ptr(), T1.data_ptr(), L.data_ptr(), n,
                                    U.data_ptr(), info.data_ptr(), st.cuda_stream)
    print('launch', n, flush=True)
    _lib.check(call())
    if os.environ.get('EIG_TRACE'):
        import time
        for _ in range(6):
            time.sleep(1.0)
            print('trace', TRACE.tolist(), flush=True)
    torch.cuda.synchronize()
    print('done', flush=True)
    r, cert, sweeps, conv = info.cpu().tolist()[:4]
    print("info", info.cpu().tolist(), flush=True)
    s, u = S.cpu().numpy(), U.cpu().numpy()
    lam_ref = np.sort(np.linalg.eigvalsh(G))[::-1]
    t_eig = timed(call)
    # the replaced path: one-sided Jacobi SVD of R^T (V accumulated), R from QR(C^T)
    R = np.linalg.qr(C.T)[1]
    B = torch.as_tensor(np.ascontiguousarray(R.T), device=dev)
    Us = torch.empty((n, n), dtype=torch.float64, device=dev)
    Ss = torch.empty(n, dtype=torch.float64, device=dev)
    Vs = torch.empty((n, n), dtype=torch.float64, device=dev)
    t_svd = timed(lambda: lib.ttk_svd_small(n, n, B.data_ptr(), Us.data_ptr(), Ss.data_ptr(), Vs.data_ptr(),
                                            st.cuda_stream))
    # truncated reconstruction vs numpy SVD
    uu, ss, vt = np.linalg.svd(C, full_matrices=False)
    ref_trunc = (uu[:, :r] * ss[:r]) @ vt[:r]
    t1, l = T1.cpu().numpy()[:, :r], L.cpu().numpy()[:, :r]
    core = t1.T @ C
    got_trunc = l @ core
    print(f"{n}x{n}: gram_eig {t_eig:.1f} us (sweeps {sweeps}, conv {conv}, r {r}, cert {cert}) vs svd_small "
          f"{t_svd:.1f} us; |S^2-eig|/l0 {np.abs(s ** 2 - lam_ref).max() / lam_ref[0]:.1e} "
          f"U orth {np.abs(u.T @ u - np.eye(n)).max():.1e} "
          f"res {np.abs(G @ u - u * s ** 2).max() / lam_ref[0]:.1e} "
          f"core orth {np.abs(core @ core.T - np.eye(r)).max():.1e} "
          f"trunc {np.linalg.norm(got_trunc - ref_trunc) / np.linalg.norm(ref_trunc):.1e}", flush=True)
