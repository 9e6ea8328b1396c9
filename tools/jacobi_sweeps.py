"""Sweep counts of one-sided Jacobi (numpy model of the GPU kernels' round-robin
order and stopping rule) on the config-3 truncation's R^T factors, with and
without cheap preconditioners.  Writes the factors to /tmp/cfg3_Bs.npy for
tools/jacobi_angle_f32.py."""
import sys, time, numpy as np
sys.path.insert(0,'/root/repo')
import oracle as O
from paper_2409_09471_b200 import configs

def jacobi_sweeps(B, skip=1e-8, order=None, maxsw=40):
    A = B.copy()
    l = A.shape[1]
    le = l + (l & 1)
    if le != l:
        A = np.concatenate([A, np.zeros((A.shape[0], 1))], axis=1)
    if order is not None:
        A = A[:, order]
    n1 = le - 1
    tol = A.shape[0] * 1.1e-16
    for sw in range(maxsw):
        big = False
        for t in range(n1):
            q = np.arange(le // 2)
            a = np.where(q == 0, t, (t + q) % n1)
            b = np.where(q == 0, n1, (t - q + n1) % n1)
            xa, xb = A[:, a], A[:, b]
            al = (xa * xa).sum(0); be = (xb * xb).sum(0); ga = (xa * xb).sum(0)
            m = (al > 0) & (be > 0) & (ga * ga > tol * tol * al * be)
            big |= np.any(ga * ga > skip * skip * al * be)
            z = np.where(m, (be - al) / (2 * np.where(m, ga, 1)), 0)
            tt = np.where(m, np.sign(z + (z == 0)) / (np.abs(z) + np.sqrt(1 + z * z)), 0)
            c = 1 / np.sqrt(1 + tt * tt); s = c * tt
            A[:, a] = c * xa - s * xb
            A[:, b] = s * xa + c * xb
        if not big:
            return sw + 1, A
    return maxsw, A

C = configs.config3()
y = O.matvec(C["op"], C["x"])
z = O.rto_sweeps(y, C["drm"])
# right-to-left truncation, collecting R^T matrices
work = [c.copy() for c in z]
d = len(work)
Bs = []
for k in range(d - 1, 0, -1):
    r0, n, r1 = work[k].shape
    M = work[k].reshape(r0, n * r1)
    q, R = np.linalg.qr(M.T)
    Bs.append(R.T.copy())
    u, s, vt = np.linalg.svd(M, full_matrices=False)
    r = min(64, len(s))
    work[k] = vt[:r].reshape(r, n, r1)
    work[k - 1] = np.tensordot(work[k - 1], u[:, :r] * s[:r], axes=([2], [0]))
np.save('/tmp/cfg3_Bs.npy', np.array(Bs))
for i in (0, 5, 15, 30):
    B = Bs[i]
    s = np.linalg.svd(B, compute_uv=False)
    print(i, "sv range", s[0], s[63] / s[0], s[-1] / s[0])
    t0 = time.time()
    n0, _ = jacobi_sweeps(B)
    n1, _ = jacobi_sweeps(B.T.copy())
    # QR step preconditioner: B^T = Q2 R2 -> Jacobi on R2^T
    R2 = np.linalg.qr(B.T)[1]
    n2, _ = jacobi_sweeps(R2.T.copy())
    # column-pivoted by norm
    nrm = (B * B).sum(0); order = np.argsort(-nrm)
    n3, _ = jacobi_sweeps(B, order=order)
    # two QR steps
    R3 = np.linalg.qr(R2.T)[1]
    n4, _ = jacobi_sweeps(R3.T.copy())
    print("  sweeps: B", n0, " B^T", n1, " QR-step", n2, " sorted", n3, " 2 QR-steps", n4, "%.1fs" % (time.time() - t0))
print("--- preconditioned by an approximate right basis")
for i in (0, 15):
    B = Bs[i]
    for prec, lab in ((np.float32, "fp32 svd"), ):
        _, _, vt = np.linalg.svd(B.astype(prec))
        V0 = vt.T.astype(np.float64)
        n5, _ = jacobi_sweeps(B @ V0)
        print(i, lab, "-> fp64 sweeps", n5)
    # approximate V from k sweeps of fp64 Jacobi without V? simulate a coarse basis: exact V perturbed
    _, _, vt = np.linalg.svd(B)
    for eps in (1e-2, 1e-3, 1e-5):
        P = vt.T + eps * np.random.default_rng(0).standard_normal(vt.shape)
        Qp = np.linalg.qr(P)[0]
        print(i, "basis err", eps, "-> sweeps", jacobi_sweeps(B @ Qp)[0])
