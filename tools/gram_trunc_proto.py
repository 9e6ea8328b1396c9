"""Prototype (numpy) of the Gram-eigen truncation step: for each core of the
left-orthogonal RTO output, G = C C^T, two-sided cyclic Jacobi (round-robin
tournament) on G, keep the top-r eigenpairs, core <- chol-orthonormalised
U_r^T C, left neighbour <- x U_r R^T.  Compares with oracle.truncate_left_orth
(the np.linalg.svd path) with the K10 metric and reports sweep counts.

usage: python tools/gram_trunc_proto.py [d] [n] [r] [ell] [cap]   (config 3: 32 128 64 80 64)
"""
import sys, os, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O
from paper_2409_09471_b200 import configs


def tournament(n):
    idx = list(range(n))
    rounds = []
    for _ in range(n - 1):
        rounds.append([(idx[i], idx[n - 1 - i]) for i in range(n // 2)])
        idx = [idx[0], idx[-1]] + idx[1:-1]
    return rounds


def jacobi_eig(G, tol=1e-8, max_sweeps=30):
    n = G.shape[0]
    G = G.copy()
    U = np.eye(n)
    rounds = tournament(n)
    sweeps = 0
    for sw in range(max_sweeps):
        rot = 0
        for pr in rounds:
            P = np.array([p for p, q in pr]); Q = np.array([q for p, q in pr])
            gpp, gqq, gpq = G[P, P], G[Q, Q], G[P, Q]
            do = np.abs(gpq) > tol * np.sqrt(gpp * gqq)
            rot += int(do.sum())
            tau = np.where(do, (gqq - gpp) / (2 * np.where(do, gpq, 1.0)), 0.0)
            t = np.where(do, np.sign(tau + (tau == 0)) / (np.abs(tau) + np.sqrt(1 + tau * tau)), 0.0)
            c = 1 / np.sqrt(1 + t * t); s = c * t
            # columns: G <- G J,  J[:, p] = c e_p - s e_q, J[:, q] = s e_p + c e_q
            gp, gq = G[:, P].copy(), G[:, Q].copy()
            G[:, P] = c * gp - s * gq; G[:, Q] = s * gp + c * gq
            gp, gq = G[P, :].copy(), G[Q, :].copy()
            G[P, :] = c[:, None] * gp - s[:, None] * gq; G[Q, :] = s[:, None] * gp + c[:, None] * gq
            up, uq = U[:, P].copy(), U[:, Q].copy()
            U[:, P] = c * up - s * uq; U[:, Q] = s * up + c * uq
        sweeps += 1
        if rot == 0:
            break
    return G, U, sweeps


def truncate_gram(cores, rel_tol=0.0, max_rank=None, tol=1e-8):
    d = len(cores)
    work = [c.copy() for c in cores]
    nrm = np.linalg.norm(work[-1])
    budget = rel_tol * nrm / np.sqrt(d - 1)
    sweeps = []
    for k in range(d - 1, 0, -1):
        r0, n, r1 = work[k].shape
        C = work[k].reshape(r0, n * r1)
        G = C @ C.T
        Gd, U, sw = jacobi_eig(G, tol)
        sweeps.append(sw)
        lam = np.diag(Gd)
        order = np.argsort(-lam)
        lam_s = lam[order]
        r = O.truncation_rank(np.sqrt(np.maximum(lam_s, 0)), budget)
        if max_rank is not None:
            r = min(r, max_rank)
        sel = order[:r]
        Ur = U[:, sel]
        Grr = Gd[np.ix_(sel, sel)]
        R = np.linalg.cholesky(Grr).T          # Grr = R^T R
        P = Ur.T @ C                           # (r x m), Gram = Grr
        newc = np.linalg.solve(R.T, P)         # R^{-T} P: orthonormal rows
        work[k] = newc.reshape(r, n, r1)
        work[k - 1] = np.tensordot(work[k - 1], Ur @ R.T, axes=([2], [0]))
    return work, sweeps


if __name__ == "__main__":
    a = [int(x) for x in sys.argv[1:]] + [None] * 5
    d, n, r, ell, cap = (a[0] or 32), (a[1] or 128), (a[2] or 64), (a[3] or 80), (a[4] or 64)
    op = configs.config3_operator(d, n, seed=0)
    x = O.gaussian_tt([n] * d, [r] * (d - 1), np.random.default_rng(1), 1.0 / np.sqrt(n * r))
    y = O.matvec(op, x)
    ls = O.rto_ranks([n] * d, [1] + [c.shape[2] for c in y], [ell] * (d - 1))
    drm = O.drm_new([n] * d, ls, seed=2)
    t0 = time.time()
    Y = O.rto_sweeps(y, drm)
    print("rto", time.time() - t0)
    t0 = time.time()
    ref = O.truncate_left_orth(Y, 0.0, cap)
    print("svd trunc", time.time() - t0)
    for tol in (1e-8, 1e-10, 1e-12):
        t0 = time.time()
        got, sw = truncate_gram(Y, 0.0, cap, tol)
        print(f"tol {tol:g}: gram trunc {time.time()-t0:.2f}s sweeps {sw} rel_diff {O.rel_diff(got, ref):.3e}",
              [c.shape[0] for c in got] == [c.shape[0] for c in ref])
