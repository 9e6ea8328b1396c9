"""numpy restatement of the reference TT hot path (TEST INFRASTRUCTURE ONLY).

All citations are to /root/reference/pkg/src/ttkrylov/<file>:<line>.  The
functions work on plain lists of float64 numpy cores:
  vector core k   : (r_{k-1}, n_k, r_k)
  operator core k : (rho_{k-1}, m_k, n_k, rho_k)
Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may use this
module; it is the checker, never the measured or shipped path.
"""

from __future__ import annotations

import math

import numpy as np

BREAKDOWN_FACTOR = 1e-14   # solvers.py:44
LSQ_RCOND = 1e-12          # solvers.py:43
CONDITION_WATERMARK = 1e-10  # solvers.py:45
PINV_RCOND = 1e-12         # streaming.py:17
ZERO_REL = 1e-14           # tt.py:355 (rounding zero test)


# ---------------------------------------------------------------------------
# constructors (tt.py:131-164, 413-447; streaming.py:38-53; sketch.py:38-47)

def attainable_ranks(dims, ranks):
    """Clip an interior rank profile to the unfolding sizes in exact integers.

    Same rule as tt.py:152-156 / streaming.py:87-90 but with Python ints, so
    it does not overflow at large d*log(n) (reference quirk Q2)."""
    d = len(dims)
    out = list(ranks)
    for k in range(1, d):
        left = math.prod(dims[:k])
        right = math.prod(dims[k:])
        out[k - 1] = int(min(out[k - 1], left, right))
    return out


def tt_random(dims, ranks, seed=0):
    """Standard-normal cores drawn k=0..d-1 from default_rng(seed) (tt.py:141-159)."""
    dims = list(dims)
    full = [1] + (attainable_ranks(dims, ranks) if len(dims) > 1 else []) + [1]
    rng = np.random.default_rng(seed)
    return [rng.standard_normal((full[k], dims[k], full[k + 1])) for k in range(len(dims))]


def gaussian_tt(dims, ranks, rng, scale=1.0):
    """Cores standard_normal((r0,n,r1)) * scale drawn in order (SURVEY 8(d) inputs)."""
    full = [1] + list(ranks) + [1]
    return [rng.standard_normal((full[k], dims[k], full[k + 1])) * scale for k in range(len(dims))]


def rank_one(vectors):
    """tt.py:136-138."""
    return [np.asarray(v, dtype=np.float64).reshape(1, -1, 1) for v in vectors]


def zero_tt(dims):
    """tt.py:131-133."""
    return [np.zeros((1, n, 1)) for n in dims]


def identity_operator(dims):
    """tt.py:162-164."""
    return [np.eye(n).reshape(1, n, n, 1) for n in dims]


def kron_sum_operator(factors):
    """Kronecker sum sum_i I x..x F_i x..x I with op-ranks 2 (tt.py:413-447).

    Channel 0 carries "factor not yet applied" ... restated: first core
    [F | I], interior [[I, 0], [F, I]], last [I ; F]."""
    mats = [np.asarray(f, dtype=np.float64) for f in factors]
    d = len(mats)
    if d == 1:
        n = mats[0].shape[0]
        return [mats[0].reshape(1, n, n, 1).copy()]
    out = []
    for i, f in enumerate(mats):
        n = f.shape[0]
        eye = np.eye(n)
        if i == 0:
            c = np.zeros((1, n, n, 2))
            c[0, :, :, 0], c[0, :, :, 1] = f, eye
        elif i == d - 1:
            c = np.zeros((2, n, n, 1))
            c[0, :, :, 0], c[1, :, :, 0] = eye, f
        else:
            c = np.zeros((2, n, n, 2))
            c[0, :, :, 0], c[1, :, :, 0], c[1, :, :, 1] = eye, f, eye
        out.append(c)
    return out


def drm_new(dims, ranks, seed=0):
    """Gaussian TT-DRM, core k ~ N(0, 1/(l_{k-1} n_k l_k)) (streaming.py:38-53)."""
    dims = list(dims)
    full = [1] + list(ranks) + [1]
    rng = np.random.default_rng(seed)
    cores = []
    for k, n in enumerate(dims):
        var = 1.0 / (full[k] * n * full[k + 1])
        cores.append(rng.normal(0.0, np.sqrt(var), size=(full[k], n, full[k + 1])))
    return cores


def kr_factors_new(dims, rows, seed=0):
    """Khatri-Rao factors with entry std rows^(-1/(2d)) (sketch.py:38-47)."""
    d = len(dims)
    std = float(rows) ** (-0.5 / d)
    rng = np.random.default_rng(seed)
    return [rng.normal(0.0, std, size=(rows, n)) for n in dims]


def frame_new(dims, recovery_ranks, oversampling=20, seed=0):
    """StreamFrame.create with exact-integer clipping (streaming.py:77-97).

    Returns (left_cores, right_cores)."""
    ranks = attainable_ranks(list(dims), list(recovery_ranks))
    lranks = [r + oversampling for r in ranks]
    s_right, s_left = np.random.SeedSequence(seed).spawn(2)
    return drm_new(dims, lranks, seed=s_left), drm_new(dims, ranks, seed=s_right)


# ---------------------------------------------------------------------------
# dense helpers (tt.py:171-200) -- small cases only

def to_dense(cores):
    acc = cores[0].reshape(cores[0].shape[1], -1)
    for c in cores[1:]:
        acc = (acc @ c.reshape(c.shape[0], -1)).reshape(-1, c.shape[2])
    return acc.reshape([c.shape[1] for c in cores])


def op_to_dense(op):
    rows, cols = op[0].shape[1], op[0].shape[2]
    acc = op[0].reshape(rows * cols, -1)
    for c in op[1:]:
        p0, mk, nk, p1 = c.shape
        acc = (acc @ c.reshape(p0, -1)).reshape(rows, cols, mk, nk, p1)
        acc = acc.transpose(0, 2, 1, 3, 4)
        rows, cols = rows * mk, cols * nk
        acc = acc.reshape(rows * cols, p1)
    return acc.reshape(rows, cols)


# ---------------------------------------------------------------------------
# exact arithmetic (tt.py:254-314)

def matvec(op, x):
    """Per-core contraction over the column index j, ranks merged as
    (a*rho0+alpha, i, b*rho1+beta) (tt.py:302-314)."""
    out = []
    for dk, ck in zip(op, x):
        p0, mk, _, p1 = dk.shape
        r0, _, r1 = ck.shape
        g = np.tensordot(ck, dk, axes=([1], [2]))          # (a, b, x, i, y)
        out.append(g.transpose(0, 2, 3, 1, 4).reshape(r0 * p0, mk, r1 * p1))
    return out


def add(a, b):
    """Block-diagonal concatenation; d == 1 adds entrywise (tt.py:254-275)."""
    d = len(a)
    if d == 1:
        return [a[0] + b[0]]
    out = []
    for k, (ca, cb) in enumerate(zip(a, b)):
        if k == 0:
            out.append(np.concatenate([ca, cb], axis=2))
        elif k == d - 1:
            out.append(np.concatenate([ca, cb], axis=0))
        else:
            ra0, n, ra1 = ca.shape
            rb0, _, rb1 = cb.shape
            blk = np.zeros((ra0 + rb0, n, ra1 + rb1))
            blk[:ra0, :, :ra1] = ca
            blk[ra0:, :, ra1:] = cb
            out.append(blk)
    return out


def scale(a, alpha):
    """The last core absorbs the factor (tt.py:278-282)."""
    out = [c.copy() for c in a]
    out[-1] *= alpha
    return out


def concat_axpy(terms, coeffs):
    """sum_t coeff_t * term_t built as tt_add(..., tt_scale(term_t, coeff_t)),
    left to right -- the explicit-mode update of solvers.py:361-366."""
    acc = scale(terms[0], coeffs[0]) if coeffs[0] != 1.0 else [c.copy() for c in terms[0]]
    for t, c in zip(terms[1:], coeffs[1:]):
        acc = add(acc, scale(t, c))
    return acc


def dot(a, b):
    """Left-to-right interface contraction (tt.py:285-294)."""
    m = np.ones((1, 1))
    for ca, cb in zip(a, b):
        t = np.tensordot(m, ca, axes=([0], [0]))       # (rb, n, ra')
        m = np.tensordot(t, cb, axes=([0, 1], [0, 1]))  # (ra', rb')
    return float(m[0, 0])


def norm(a):
    """tt.py:297-299."""
    return float(np.sqrt(max(dot(a, a), 0.0)))


# ---------------------------------------------------------------------------
# TT-SVD rounding (tt.py:203-211, 321-368)

def truncation_rank(sv, budget):
    """Smallest r whose discarded tail ||sv[r:]|| <= budget, at least 1 (tt.py:203-211)."""
    sv = np.asarray(sv)
    if sv.size == 0:
        return 1
    tail = np.sqrt(np.maximum(np.cumsum(sv[::-1] ** 2)[::-1], 0.0))
    hit = np.flatnonzero(tail <= budget)
    r = int(hit[0]) if hit.size else sv.size
    return max(r, 1)


def right_orthogonalize(cores):
    """R->L Householder QR sweep; the norm ends in core 0 (tt.py:321-334)."""
    cores = list(cores)
    for k in range(len(cores) - 1, 0, -1):
        r0, n, r1 = cores[k].shape
        q, lt = np.linalg.qr(cores[k].reshape(r0, n * r1).T)
        cores[k] = q.T.reshape(q.shape[1], n, r1)
        cores[k - 1] = np.tensordot(cores[k - 1], lt.T, axes=([2], [0]))
    return cores


def tt_round(cores, rel_tol=0.0, max_rank=None, zero_rel=ZERO_REL):
    """TT-SVD recompression (tt.py:337-368).

    zero_rel=ZERO_REL keeps the reference's cancellation test (tt.py:348-356);
    zero_rel=None disables it (reference quirk Q1)."""
    d = len(cores)
    if d == 1:
        return [cores[0].copy()]
    prod_scale = 1.0
    if zero_rel is not None:
        with np.errstate(over="ignore"):
            for c in cores:
                prod_scale *= np.linalg.norm(c)
    work = right_orthogonalize([c.copy() for c in cores])
    nrm = np.linalg.norm(work[0])
    if nrm == 0 or (zero_rel is not None and nrm <= zero_rel * prod_scale):
        return zero_tt([c.shape[1] for c in cores])
    budget = rel_tol * nrm / np.sqrt(d - 1)
    for k in range(d - 1):
        r0, n, r1 = work[k].shape
        u, sv, vt = np.linalg.svd(work[k].reshape(r0 * n, r1), full_matrices=False)
        r = truncation_rank(sv, budget)
        if max_rank is not None:
            r = min(r, max_rank)
        work[k] = u[:, :r].reshape(r0, n, r)
        work[k + 1] = np.tensordot(sv[:r, None] * vt[:r], work[k + 1], axes=([1], [0]))
    return work


# ---------------------------------------------------------------------------
# randomize-then-orthogonalize (absent from the reference, SPEC.md:313;
# restated from PAPER.md:435-445 and SURVEY.md Appendix B)

def rto_ranks(dims, in_ranks, ell):
    """Sketch ranks l_c (c = 1..d-1): min(ell_c, R_c, attainable), then
    l_c <= l_{c-1} * n_{c-1} so every QR below is tall."""
    d = len(dims)
    if np.isscalar(ell):
        ell = [int(ell)] * (d - 1)
    ls = [int(min(e, r)) for e, r in zip(ell, in_ranks[1:-1])]
    ls = attainable_ranks(list(dims), ls)
    prev = 1
    for c in range(d - 1):
        ls[c] = max(1, min(ls[c], prev * dims[c]))
        prev = ls[c]
    return ls


def slice_drm(drm, ls):
    """Leading slices of a DRM drawn at a larger rank profile."""
    full = [1] + list(ls) + [1]
    return [g[: full[k], :, : full[k + 1]] for k, g in enumerate(drm)]


def rto_sweeps(cores, drm):
    """Randomize-then-orthogonalize: right partial contractions with the
    Gaussian TT `drm`, then the left-to-right sketch/QR/project sweep.
    Returns left-orthogonal cores with ranks given by the DRM."""
    d = len(cores)
    if d == 1:
        return [cores[0].copy()]
    # step 1: W_c (R_c x l_c), right partial contractions, streaming.py:133-136 recurrence
    w = [None] * (d + 1)
    w[d] = np.ones((1, 1))
    for c in range(d - 1, 0, -1):
        r0, n, r1 = cores[c].shape
        t = (cores[c].reshape(r0 * n, r1) @ w[c + 1]).reshape(r0, n * w[c + 1].shape[1])
        g = drm[c]
        w[c] = t @ g.reshape(g.shape[0], -1).T
    # step 2: left sweep
    out = []
    z = cores[0].reshape(-1, cores[0].shape[2])  # (l_{c-1} n_{c-1}) x R_c
    for c in range(1, d):
        y = z @ w[c]
        q, _ = np.linalg.qr(y)
        lc = q.shape[1]
        out.append(q.reshape(-1, cores[c - 1].shape[1], lc))
        mproj = q.T @ z                                      # l_c x R_c
        nxt = cores[c]
        z = (mproj @ nxt.reshape(nxt.shape[0], -1)).reshape(lc * nxt.shape[1], nxt.shape[2])
    out.append(z.reshape(-1, cores[d - 1].shape[1], 1))
    return out


def truncate_left_orth(cores, rel_tol=0.0, max_rank=None):
    """TT-SVD truncation of a LEFT-orthogonal TT, right to left.

    For a TT whose cores 0..d-2 are left-orthonormal (the RTO output) the
    norm sits in the last core and the right unfoldings of the cores carry the
    singular values of the tensor's unfoldings, so the TT-SVD needs no
    orthogonalisation sweep: for k = d-1..1 take the SVD of C_k as
    (r_{k-1} x n_k r_k), keep the _truncation_rank (tt.py:203-211) with the
    budget rel_tol ||v|| / sqrt(d-1) (tt.py:357) and the cap, keep V^T in C_k and
    absorb U S into C_{k-1}."""
    d = len(cores)
    work = [c.copy() for c in cores]
    if d == 1:
        return work
    nrm = np.linalg.norm(work[-1])
    if nrm == 0:
        return zero_tt([c.shape[1] for c in cores])
    budget = rel_tol * nrm / np.sqrt(d - 1)
    for k in range(d - 1, 0, -1):
        r0, n, r1 = work[k].shape
        u, sv, vt = np.linalg.svd(work[k].reshape(r0, n * r1), full_matrices=False)
        r = truncation_rank(sv, budget)
        if max_rank is not None:
            r = min(r, max_rank)
        work[k] = vt[:r].reshape(r, n, r1)
        work[k - 1] = np.tensordot(work[k - 1], u[:, :r] * sv[None, :r], axes=([2], [0]))
    return work


def rto_round(cores, drm, rel_tol=0.0, max_rank=None):
    """Randomized rounding: RTO sweeps, then the right-to-left TT-SVD
    truncation of the left-orthogonal result."""
    return truncate_left_orth(rto_sweeps(cores, drm), rel_tol, max_rank)


def rto_flops(dims, in_ranks, ls):
    """Algorithmic FLOPs of rto_sweeps (SURVEY 8(d) formula, QR as 4ml^2-4l^3/3)."""
    d = len(dims)
    L = [1] + list(ls) + [1]
    R = list(in_ranks)
    f = 0.0
    for c in range(d - 1, 0, -1):  # right sweep, core c
        n = dims[c]
        f += 2.0 * R[c] * n * R[c + 1] * L[c + 1] + 2.0 * R[c] * n * L[c + 1] * L[c]
    for c in range(1, d):  # left sweep, cut c
        m = L[c - 1] * dims[c - 1]
        l = L[c]
        f += 2.0 * m * R[c] * l + (4.0 * m * l * l - 4.0 * l ** 3 / 3.0) + 2.0 * l * m * R[c]
        f += 2.0 * l * R[c] * dims[c] * R[c + 1]
    return f


def matvec_flops(op_shapes, x_ranks):
    """Dense matvec FLOPs: sum_k 2 rho0 m n rho1 r0 r1."""
    f = 0.0
    for (p0, m, n, p1), r0, r1 in zip(op_shapes, x_ranks[:-1], x_ranks[1:]):
        f += 2.0 * p0 * m * n * p1 * r0 * r1
    return f


# ---------------------------------------------------------------------------
# Khatri-Rao sketch (sketch.py:50-70)

def kr_apply(factors, cores):
    """Row-wise running state over the modes: state <- state x (F_k[j] . C_k)."""
    rows = factors[0].shape[0]
    state = np.ones((rows, 1))
    for f, c in zip(factors, cores):
        mk = np.tensordot(f, c, axes=([1], [1]))  # (rows, r0, r1)
        state = np.einsum("sa,sab->sb", state, mk)
    return state[:, 0].copy()


def kr_flops(rows, dims, ranks):
    return sum(2.0 * rows * n * r0 * r1 for n, r0, r1 in zip(dims, ranks[:-1], ranks[1:]))


# ---------------------------------------------------------------------------
# streaming sketches (streaming.py:117-205)

def stream_sketch(cores, left, right):
    """Psi/Omega of one tensor against a frame (streaming.py:117-142).

    left/right: Y (oversampled) and X (recovery) DRM cores."""
    d = len(cores)
    lm = [np.ones((1, 1))]
    for k in range(d - 1):
        y, c = left[k], cores[k]
        t = np.tensordot(lm[k], c, axes=([1], [0]))            # (l, n, t')
        lm.append(np.tensordot(y, t, axes=([0, 1], [0, 1])))  # (l', t')
    rm = [None] * (d + 1)
    rm[d] = np.ones((1, 1))
    for k in range(d - 1, 0, -1):
        c, x = cores[k], right[k]
        t = np.tensordot(c, rm[k + 1], axes=([2], [0]))         # (t, n, r')
        rm[k] = np.tensordot(t, x, axes=([1, 2], [1, 2]))      # (t, r)
    psi = []
    for mu in range(d):
        p = np.tensordot(lm[mu], cores[mu], axes=([1], [0]))   # (l, n, t')
        p = np.tensordot(p, rm[mu + 1], axes=([2], [0]))       # (l, n, r)
        psi.append(p.reshape(-1, p.shape[2]))
    omega = [lm[mu] @ rm[mu] for mu in range(1, d)]
    return psi, omega


def combine_pairs(pairs, coeffs):
    """Entrywise weighted sum, first term scaled then accumulated (streaming.py:145-163)."""
    psi = [c * coeffs[0] for c in pairs[0][0]]
    omega = [c * coeffs[0] for c in pairs[0][1]]
    for (ps, om), a in zip(pairs[1:], coeffs[1:]):
        for k, m in enumerate(ps):
            psi[k] += a * m
        for k, m in enumerate(om):
            omega[k] += a * m
    return psi, omega


def stream_recover(psi, omega, dims, rel_tol=0.0, max_rank=None, zero_rel=ZERO_REL):
    """Generalised-Nystrom core recovery with symmetric S^{-1/2} split of
    pinv(Omega_mu) (rcond PINV_RCOND), then tt_round (streaming.py:166-205)."""
    d = len(psi)
    if all(not np.any(p) for p in psi):
        return zero_tt(dims)
    lh, rh = [], []
    for mu, om in enumerate(omega):
        if not np.any(om):
            raise ValueError(f"zero cross matrix at mode {mu + 1}")
        u, sv, vt = np.linalg.svd(om, full_matrices=False)
        keep = sv > PINV_RCOND * sv[0]
        u, sv, vt = u[:, keep], sv[keep], vt[keep]
        s = 1.0 / np.sqrt(sv)
        lh.append(s[:, None] * u.T)
        rh.append(vt.T * s[None, :])
    cores = []
    for mu in range(d):
        p = psi[mu]
        n = dims[mu]
        blk = p.reshape(p.shape[0] // n, n, p.shape[1])
        if mu > 0:
            blk = np.tensordot(lh[mu - 1], blk, axes=([1], [0]))
        if mu < d - 1:
            blk = np.tensordot(blk, rh[mu], axes=([2], [0]))
        cores.append(blk)
    return tt_round(cores, rel_tol, max_rank, zero_rel=zero_rel)


# ---------------------------------------------------------------------------
# solver (solvers.py:119-155, 334-465)

def lsq_svd(w, rhs):
    """np.linalg.lstsq with rcond 1e-12 and the explicit residual (solvers.py:129-134)."""
    y, _, _, sv = np.linalg.lstsq(w, rhs, rcond=LSQ_RCOND)
    return y, float(np.linalg.norm(w @ y - rhs)), sv


def solution_rank(b_ranks, cfg):
    """solvers.py:144-147."""
    if cfg.get("solution_rank") is not None:
        return cfg["solution_rank"]
    return max(max(b_ranks) * 2, 20)


def solver_frame(b, cfg, seed):
    """make_solver_frame without the cumprod overflow (solvers.py:150-155, quirk Q2)."""
    sol = solution_rank([1] + [c.shape[2] for c in b], cfg)
    ranks = [max(c.shape[2], 2 * sol) for c in b[:-1]]
    return frame_new([c.shape[1] for c in b], ranks, cfg.get("oversampling", 20), seed)


def sgmres(op, b, cfg, factors, frame=None, rounding="svd", rto_drm=None, precond=None):
    """TT-sGMRES with sketch-only basis memory (solvers.py:334-431, 450-480).

    cfg keys: maxit, tol, ell, eta, max_rank, oversampling, solution_rank,
    combine_mode ('explicit'|'stta'), seed, zero_rel.  rounding='svd' uses
    tt_round (TT-SVD); rounding='rto' uses rto_round with one DRM per solve
    (rto_drm, drawn at the maximal sketch-rank profile, leading slices reused).
    precond: optional callable cores -> cores, the right preconditioner P^{-1}
    of tt_spgmres (solvers.py:315-320, 462-463, 483-490).
    x0 is taken as zero.  Returns (x_cores, report_dict)."""
    maxit, tol, ell = cfg["maxit"], cfg["tol"], cfg["ell"]
    eta, max_rank = cfg.get("eta", 0.3), cfg.get("max_rank")
    zero_rel = cfg.get("zero_rel", ZERO_REL)
    mode = cfg.get("combine_mode", "explicit")
    dims = [c.shape[1] for c in b]
    if frame is None:
        frame = solver_frame(b, cfg, cfg.get("seed", 0) + 1)
    left, right = frame

    def rnd(v, rel, cap):
        if rounding == "svd":
            return tt_round(v, rel, cap, zero_rel=zero_rel)
        rk = [1] + [c.shape[2] for c in v]
        ls = rto_ranks(dims, rk, [g.shape[2] for g in rto_drm[:-1]])
        return rto_round(v, slice_drm(rto_drm, ls), rel, cap)

    rep = {"res_sketched": [], "basis_rank": [], "iterations": 0, "converged": False,
           "max_resident_basis": 0, "warnings": [], "h": []}
    nb_sketch = float(np.linalg.norm(kr_apply(factors, b)))
    beta = norm(b)
    if beta == 0 or nb_sketch == 0:
        rep["converged"] = True
        return [c.copy() for c in b], rep
    v1 = scale(b, 1.0 / beta)
    sr0 = kr_apply(factors, b)
    pairs = [stream_sketch(v1, left, right)]
    window = [(0, v1)]
    wcols = []
    y = np.zeros(1)
    for k in range(1, maxit + 1):
        vt = window[-1][1]
        if precond is not None:
            vt = precond(vt)
        vt = matvec(op, vt)
        norm_av = norm(vt)
        wcols.append(kr_apply(factors, vt))
        if mode == "explicit":
            hs = []
            for gi, vi in window:
                hik = dot(vt, vi)
                hs.append(hik)
                vt = add(vt, scale(vi, -hik))
            vt = rnd(vt, eta * tol, max_rank)
        else:
            hs = [dot(vt, vi) for _, vi in window]
            pv = stream_sketch(vt, left, right)
            comb = combine_pairs([pv] + [pairs[gi] for gi, _ in window], [1.0] + [-h for h in hs])
            vt = stream_recover(comb[0], comb[1], dims, eta * tol, max_rank, zero_rel=zero_rel)
        rep["h"].append(hs)
        hnew = norm(vt)
        lucky = hnew <= BREAKDOWN_FACTOR * norm_av
        if not lucky:
            vnew = scale(vt, 1.0 / hnew)
            pairs.append(stream_sketch(vnew, left, right))
            rep["max_resident_basis"] = max(rep["max_resident_basis"], len(window) + 1)
            window.append((k, vnew))
            if len(window) > ell:
                window.pop(0)
        w = np.stack(wcols, axis=1)
        y, res, sv = lsq_svd(w, sr0)
        if sv.size and sv[-1] < CONDITION_WATERMARK * sv[0]:
            msg = f"iteration {k}: sketched basis nearly rank-deficient"
            if not rep["warnings"] or rep["warnings"][-1][:9] != msg[:9]:
                rep["warnings"].append(msg)
        rep["res_sketched"].append(res / nb_sketch)
        rep["basis_rank"].append(max((max([1] + [c.shape[2] for c in v]) for _, v in window), default=1))
        rep["iterations"] = k
        hit = res <= nb_sketch * tol
        if hit:
            rep["converged"] = True
        if hit or lucky:
            if lucky:
                rep["converged"] = True
            break
    ps = [pairs[i] for i in range(len(y))]
    comb = combine_pairs(ps, [float(c) for c in y])
    x = stream_recover(comb[0], comb[1], dims, tol, solution_rank([1] + [c.shape[2] for c in b], cfg),
                       zero_rel=zero_rel)
    if precond is not None:
        x = precond(x)
    rep["y"] = np.asarray(y)
    return x, rep


# ---------------------------------------------------------------------------
# exp-sum preconditioner apply (precond.py:189-200, 246-278)

def mode_multiply(cores, mats):
    """O_k[a, i, b] = sum_j M_k[i, j] C_k[a, j, b]; ranks unchanged (precond.py:189-200)."""
    return [np.einsum("ij,ajb->aib", np.asarray(m, dtype=np.float64), c) for m, c in zip(mats, cores)]


def expsum_apply(cores, exps, alpha, rel_tol, max_rank=None, accumulate="sequential", frame=None,
                 zero_rel=ZERO_REL):
    """sum_j alpha_j (x_i exp(-beta_j A_i)) v accumulated by rounded additions
    (inner rounding without rank cap, final with cap) or in sketch space
    against ``frame`` = (left, right) DRM cores (precond.py:246-278).
    exps[j][k] = exp(-beta_j A_k)."""
    terms = [scale(mode_multiply(cores, exps[j]), float(alpha[j])) for j in range(len(alpha))]
    if accumulate == "sequential":
        acc = terms[0]
        for t in terms[1:]:
            acc = tt_round(add(acc, t), rel_tol, None, zero_rel=zero_rel)
        return tt_round(acc, rel_tol, max_rank, zero_rel=zero_rel)
    left, right = frame
    psi, omega = combine_pairs([stream_sketch(t, left, right) for t in terms], [1.0] * len(terms))
    return stream_recover(psi, omega, [c.shape[1] for c in cores], rel_tol, max_rank, zero_rel=zero_rel)


def true_residual(op, b, x, zero_rel=ZERO_REL):
    """||b - A x|| / ||b|| with one rounding at 1e-12 (solvers.py:137-141)."""
    r = tt_round(add(b, scale(matvec(op, x), -1.0)), 1e-12, None, zero_rel=zero_rel)
    nb = norm(b)
    return norm(r) / nb if nb > 0 else norm(r)


# ---------------------------------------------------------------------------
# parity metric: orthogonalise the difference, then ||core0||

def diff_norm(a, b):
    """||a - b|| resolved below 1e-14 by right-orthogonalising the difference."""
    diff = add(a, scale(b, -1.0))
    if len(diff) == 1:
        return float(np.linalg.norm(diff[0]))
    return float(np.linalg.norm(right_orthogonalize(diff)[0]))


def orth_norm(a):
    """||a|| from the right-orthogonalised core 0 (no dot-product cancellation)."""
    if len(a) == 1:
        return float(np.linalg.norm(a[0]))
    return float(np.linalg.norm(right_orthogonalize([c.copy() for c in a])[0]))


def rel_diff(a, b):
    """||a - b|| / ||b|| with the K10 metric."""
    return diff_norm(a, b) / max(orth_norm(b), 1e-300)
