"""Seeded synthetic inputs of the five BASELINE.json configurations.

All Gaussian draws use numpy default_rng on the host (SURVEY.md 8(d)
"Canonical inputs"), so the GPU path and the CPU oracle see identical data.
The builders return plain numpy cores; callers upload them.
"""

from __future__ import annotations

import math

import numpy as np


def tridiag(n, sub, diag, sup):
    return np.diag(np.full(n, diag)) + np.diag(np.full(n - 1, sub), -1) + np.diag(np.full(n - 1, sup), 1)


def kron_sum_cores(mats):
    """op-rank-2 Kronecker-sum cores (reference tt.py:413-447)."""
    d = len(mats)
    out = []
    for i, f in enumerate(mats):
        n = f.shape[0]
        eye = np.eye(n)
        if d == 1:
            out.append(f.reshape(1, n, n, 1).copy())
        elif i == 0:
            c = np.zeros((1, n, n, 2)); c[0, :, :, 0], c[0, :, :, 1] = f, eye; out.append(c)
        elif i == d - 1:
            c = np.zeros((2, n, n, 1)); c[0, :, :, 0], c[1, :, :, 0] = eye, f; out.append(c)
        else:
            c = np.zeros((2, n, n, 2)); c[0, :, :, 0], c[1, :, :, 0], c[1, :, :, 1] = eye, f, eye
            out.append(c)
    return out


def gaussian_tt(dims, ranks, rng, scale):
    full = [1] + list(ranks) + [1]
    return [rng.standard_normal((full[k], dims[k], full[k + 1])) * scale for k in range(len(dims))]


def concat_cores(a, b):
    """Block-diagonal TT sum (reference tt_add, tt.py:254-275), host side."""
    d = len(a)
    out = []
    for k, (ca, cb) in enumerate(zip(a, b)):
        if k == 0:
            out.append(np.concatenate([ca, cb], axis=2))
        elif k == d - 1:
            out.append(np.concatenate([ca, cb], axis=0))
        else:
            blk = np.zeros((ca.shape[0] + cb.shape[0], ca.shape[1], ca.shape[2] + cb.shape[2]))
            blk[: ca.shape[0], :, : ca.shape[2]] = ca
            blk[ca.shape[0]:, :, ca.shape[2]:] = cb
            out.append(blk)
    return out


def drm_cores(dims, ranks, seed):
    """reference tt_drm_new (streaming.py:38-53) draws."""
    full = [1] + list(ranks) + [1]
    rng = np.random.default_rng(seed)
    return [rng.normal(0.0, np.sqrt(1.0 / (full[k] * n * full[k + 1])), size=(full[k], n, full[k + 1]))
            for k, n in enumerate(dims)]


# ---------------------------------------------------------------------------

def config1():
    """TT-sGMRES, d=8, n=32 Laplacian (op-rank 2), rank-1 normalised RHS."""
    n, d = 32, 8
    lap = (n + 1) ** 2 * tridiag(n, -1.0, 2.0, -1.0)
    op = kron_sum_cores([lap] * d)
    rng = np.random.default_rng(0)
    vecs = [rng.standard_normal(n) for _ in range(d)]
    b = [v.reshape(1, n, 1) for v in vecs]
    nb = math.prod(float(np.linalg.norm(v)) for v in vecs)
    b[-1] = b[-1] / nb
    cfg = dict(maxit=40, tol=1e-8, ell=2, eta=1.0, max_rank=30, sketch_rows=80, seed=0)
    return {"op": op, "b": b, "cfg": cfg, "sketch_seed": 0, "frame_seed": 1, "dims": [n] * d}


def config2():
    """Randomized rounding microbench: sum of 10 rank-20 TTs (d=16, n=64) -> rank 200."""
    d, n, r = 16, 64, 20
    rng = np.random.default_rng(0)
    terms = [gaussian_tt([n] * d, [r] * (d - 1), rng, 1.0 / math.sqrt(n * r)) for _ in range(10)]
    x = terms[0]
    for t in terms[1:]:
        x = concat_cores(x, t)
    drm = drm_cores([n] * d, [50] * (d - 1), seed=1)
    return {"x": x, "drm": drm, "ell": 50, "max_rank": 40, "rel_tol": 0.0, "dims": [n] * d}


def config3_operator(d=32, n=128, seed=0):
    """Explicit 3-channel anisotropic convection-diffusion operator:
    first [I, c_1 L, B]; interior [[I, c_k L, B], [0, I, 0], [0, 0, I]]; last [c_d L + B; I; I]."""
    c = np.random.default_rng(seed).uniform(0.1, 1.0, d)
    h = 1.0 / (n + 1)
    lap = tridiag(n, -1.0, 2.0, -1.0) / h ** 2
    conv = tridiag(n, -1.0, 0.0, 1.0) / (2 * h)
    eye = np.eye(n)
    cores = []
    for k in range(d):
        if k == 0:
            g = np.zeros((1, n, n, 3)); g[0, :, :, 0], g[0, :, :, 1], g[0, :, :, 2] = eye, c[k] * lap, conv
        elif k == d - 1:
            g = np.zeros((3, n, n, 1)); g[0, :, :, 0], g[1, :, :, 0], g[2, :, :, 0] = c[k] * lap + conv, eye, eye
        else:
            g = np.zeros((3, n, n, 3))
            g[0, :, :, 0], g[0, :, :, 1], g[0, :, :, 2] = eye, c[k] * lap, conv
            g[1, :, :, 1], g[2, :, :, 2] = eye, eye
        cores.append(g)
    return cores


def config3():
    """matvec (rho=3, r=64 -> 192) + randomized rounding l=80 -> 64, d=32, n=128."""
    d, n, r = 32, 128, 64
    op = config3_operator(d, n, seed=0)
    x = gaussian_tt([n] * d, [r] * (d - 1), np.random.default_rng(1), 1.0 / math.sqrt(n * r))
    drm = drm_cores([n] * d, [80] * (d - 1), seed=2)
    return {"op": op, "x": x, "drm": drm, "ell": 80, "max_rank": 64, "rel_tol": 0.0, "dims": [n] * d}


def config4(nvec=64):
    """Khatri-Rao sketch, s=512 rows, N(0,1/n) factors, 64 TTs d=20, n=64, r=100."""
    d, n, r, s = 20, 64, 100, 512
    rng = np.random.default_rng(0)
    factors = [rng.normal(0.0, 1.0 / math.sqrt(n), size=(s, n)) for _ in range(d)]
    rng = np.random.default_rng(1)
    vecs = [gaussian_tt([n] * d, [r] * (d - 1), rng, 1.0 / math.sqrt(n * r)) for _ in range(nvec)]
    return {"factors": factors, "vecs": vecs, "rows": s, "dims": [n] * d}


def config5(rhs_index=0):
    """TT-sGMRES, d=50, n=256 anisotropic Laplacian (op-rank 2), RHS j = rank-1 from rng(j)."""
    d, n = 50, 256
    c = np.random.default_rng(0).uniform(0.1, 1.0, d)
    lap = (n + 1) ** 2 * tridiag(n, -1.0, 2.0, -1.0)
    op = kron_sum_cores([ck * lap for ck in c])
    rng = np.random.default_rng(rhs_index)
    vecs = [rng.standard_normal(n) for _ in range(d)]
    b = [v.reshape(1, n, 1) for v in vecs]
    nb = math.prod(float(np.linalg.norm(v)) for v in vecs)
    b[-1] = b[-1] / nb
    cfg = dict(maxit=60, tol=1e-8, ell=3, eta=1.0, max_rank=100, sketch_rows=120, seed=rhs_index)
    return {"op": op, "b": b, "cfg": cfg, "sketch_seed": rhs_index, "frame_seed": rhs_index + 1,
            "dims": [n] * d}


def matvec_flops(op, ranks):
    return sum(2.0 * g.shape[0] * g.shape[1] * g.shape[2] * g.shape[3] * ranks[k] * ranks[k + 1]
               for k, g in enumerate(op))


def kr_flops(rows, dims, ranks):
    return sum(2.0 * rows * n * r0 * r1 for n, r0, r1 in zip(dims, ranks[:-1], ranks[1:]))
