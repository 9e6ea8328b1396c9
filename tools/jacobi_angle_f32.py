"""Jacobi with the rotation angle computed in fp32 and (c, s) renormalised in fp64: sweep counts and accuracy (numpy model)."""
import numpy as np, sys
sys.path.insert(0,'/tmp/jx')
Bs = np.load('/tmp/cfg3_Bs.npy')  # written by tools/jacobi_sweeps.py

def jac(B, f32angle, skip=1e-8, maxsw=40):
    A = B.copy(); l = A.shape[1]; le = l; n1 = le - 1
    V = np.eye(l)
    tol = A.shape[0] * 1.1e-16
    for sw in range(maxsw):
        big = False
        for t in range(n1):
            q = np.arange(le // 2)
            a = np.where(q == 0, t, (t + q) % n1); b = np.where(q == 0, n1, (t - q + n1) % n1)
            xa, xb = A[:, a], A[:, b]
            al = (xa * xa).sum(0); be = (xb * xb).sum(0); ga = (xa * xb).sum(0)
            m = (al > 0) & (be > 0) & (ga * ga > tol * tol * al * be)
            big |= np.any(ga * ga > skip * skip * al * be)
            sc = 1.0 / (al + be)
            dd = (be - al) * sc; w = 2 * ga * sc
            if f32angle:
                df = dd.astype(np.float32); wf = w.astype(np.float32)
                qf = df * df + wf * wf
                rf = np.sqrt(qf); sf = np.abs(df) + rf
                rqf = (1 / np.sqrt(2 * rf * sf)).astype(np.float32)
                c0 = (sf * rqf).astype(np.float64); s0 = (np.where(df >= 0, wf, -wf) * rqf).astype(np.float64)
                dl = c0 * c0 + s0 * s0 - 1
                f = 1 + dl * (-0.5 + 0.375 * dl)
                c = c0 * f; s = s0 * f
            else:
                qq = dd * dd + w * w; rho = np.sqrt(qq); sm = np.abs(dd) + rho
                rq = 1 / np.sqrt(2 * rho * sm)
                c = sm * rq; s = np.where(dd >= 0, w, -w) * rq
            c = np.where(m, c, 1.0); s = np.where(m, s, 0.0)
            A[:, a] = c * xa - s * xb; A[:, b] = s * xa + c * xb
            va, vb = V[:, a], V[:, b]
            V[:, a] = c * va - s * vb; V[:, b] = s * va + c * vb
        if not big:
            return sw + 1, A, V
    return maxsw, A, V

for i in (0, 15, 30):
    B = Bs[i]
    s0 = np.linalg.svd(B, compute_uv=False)
    for f in (False, True):
        n, A, V = jac(B, f)
        nr = np.sqrt((A * A).sum(0)); U = A / nr
        print(i, "f32angle" if f else "fp64angle", "sweeps", n, "U orth %.1e V orth %.1e sv err %.1e res %.1e" % (
            np.abs(U.T @ U - np.eye(80)).max(), np.abs(V.T @ V - np.eye(80)).max(),
            np.max(np.abs(np.sort(nr)[::-1] - s0) / s0), np.linalg.norm(B @ V - A) / np.linalg.norm(B)))
