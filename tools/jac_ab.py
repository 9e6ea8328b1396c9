"""Jacobi SVD timing + accuracy at in-step sizes (run with and without
TTK_JACOBI_SINGLE=1 to compare the cluster and single-CTA kernels)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2409_09471_b200 import _lib

lib = _lib.load()
dev = torch.device("cuda", 0)
st = _lib.stream_ptr(dev)
cnt = torch.zeros(1, dtype=torch.int32, device=dev)
rng = np.random.default_rng(0)


def ev_time(fn, reps=20):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); [fn() for _ in range(reps)]; b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


res = {"mode": "single" if os.environ.get("TTK_JACOBI_SINGLE") else "cluster"}
for kind in ("gauss", "graded"):
    for k in (7, 20, 33, 50, 80, 100, 128):
        A = rng.standard_normal((4 * k, k))
        if kind == "graded":
            A = A * np.logspace(0, -12, k)[None, :]
        R = np.linalg.qr(A)[1]
        Bt = np.ascontiguousarray(R.T)  # the R^T variant used in rounding
        B = torch.as_tensor(Bt, device=dev)
        U = torch.empty((k, k), dtype=torch.float64, device=dev)
        S = torch.empty(k, dtype=torch.float64, device=dev)
        V = torch.empty((k, k), dtype=torch.float64, device=dev)
        lib.ttk_debug_svd_sweeps(cnt.data_ptr())
        rc = lib.ttk_svd_small(k, k, B.data_ptr(), U.data_ptr(), S.data_ptr(), V.data_ptr(), st)
        if rc != 0:
            res[f"{kind}_{k}"] = {"error": lib.ttk_last_error().decode()}
            lib.ttk_debug_svd_sweeps(None)
            continue
        torch.cuda.synchronize()
        sweeps = int(cnt.item())
        lib.ttk_debug_svd_sweeps(None)
        prof = torch.zeros(40, dtype=torch.int64, device=dev)
        lib.ttk_debug_jacobi_profile(prof.data_ptr())
        lib.ttk_svd_small(k, k, B.data_ptr(), U.data_ptr(), S.data_ptr(), V.data_ptr(), st)
        torch.cuda.synchronize()
        lib.ttk_debug_jacobi_profile(None)
        pr = prof.view(8, 5).cpu().numpy()
        phases = [round(float(v), 1) for v in (pr[0, :4] / max(pr[0, 4], 1))]
        us = ev_time(lambda: lib.ttk_svd_small(k, k, B.data_ptr(), U.data_ptr(), S.data_ptr(), V.data_ptr(), st))
        u, s, v = U.cpu().numpy(), S.cpu().numpy(), V.cpu().numpy()
        sref = np.linalg.svd(Bt, compute_uv=False)
        rec = np.abs(Bt @ v - u * s[None, :]).max() / sref[0]
        orth_v = np.abs(v.T @ v - np.eye(k)).max()
        keep = s > 1e-10 * s[0]
        orth_u = np.abs(u[:, keep].T @ u[:, keep] - np.eye(int(keep.sum()))).max()
        res[f"{kind}_{k}"] = {"us": round(us, 1), "sweeps": sweeps, "cyc_per_round_cta0": phases,
                              "sv_rel": float(np.abs(s - sref).max() / sref[0]),
                              "rec": float(rec), "orth_v": float(orth_v), "orth_u": float(orth_u)}
print(json.dumps(res))
