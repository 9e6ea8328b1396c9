"""Exp-sum preconditioner on the device (ttk_mode_multiply + device rounding /
streaming) and right-preconditioned tt_spgmres, against the reference's own
outputs (golden/precond.npz) and the oracle."""

import numpy as np
import pytest
import torch

import oracle as O
import paper_2409_09471_b200 as T
from paper_2409_09471_b200 import precond as P
from golden_io import cores, factors, load

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def z():
    return load("precond.npz")


def _lap(n):
    return -(-2.0 * np.eye(n) + np.diag(np.ones(n - 1), 1) + np.diag(np.ones(n - 1), -1))


def _dense(v):
    return T.tt_to_dense(v).cpu().numpy()


def _rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b)


def test_mode_multiply_golden(cuda, z):
    """Rectangular mode matrices (mode sizes change), against the reference's mode_multiply."""
    v = T.TTVector(cores(z, "mm_in"), device=cuda)
    w = T.mode_multiply(v, [z[f"mm_mat{k}"] for k in range(3)])
    assert w.ranks == v.ranks and w.dims == (5, 4, 2)
    for g, want in zip(w.cores, cores(z, "mm_out")):
        assert np.abs(g.cpu().numpy() - want).max() <= 1e-14 * np.abs(want).max()


def test_mode_multiply_many_terms_vs_oracle(cuda):
    """17 terms x 8 cores = 136 products (two grouped launches), ragged ranks,
    alpha on the last core; each term against the oracle."""
    rng = np.random.default_rng(3)
    dims, ranks = [7, 16, 33, 5, 64, 9, 12, 20], [1, 7, 40, 13, 5, 60, 9, 17, 1]
    xc = [rng.standard_normal((ranks[k], dims[k], ranks[k + 1])) for k in range(8)]
    mats = [[rng.standard_normal((dims[k], dims[k])) for k in range(8)] for _ in range(17)]
    alpha = rng.standard_normal(17)
    v = T.TTVector(xc, device=cuda)
    dm = [[torch.as_tensor(m, device=cuda) for m in row] for row in mats]
    outs = P._mode_multiply_many(v, dm, list(alpha))
    for t in range(17):
        want = O.scale(O.mode_multiply(xc, mats[t]), alpha[t])
        for g, w in zip(outs[t].cores, want):
            assert np.abs(g.cpu().numpy() - w).max() <= 1e-13 * np.abs(w).max()


def test_mode_multiply_errors(cuda):
    v = T.TTVector([np.ones((1, 3, 2)), np.ones((2, 4, 1))], device=cuda)
    with pytest.raises(T.ShapeMismatch):
        T.mode_multiply(v, [np.eye(3)])
    with pytest.raises(T.ShapeMismatch):
        T.mode_multiply(v, [np.eye(3), np.eye(5)])


def test_precond_apply_golden(cuda, z):
    """Approximate inverse of a 3-mode Laplacian, zeta 24 (test_precond.py:145-156)."""
    fac = [_lap(6)] * 3
    # coefficients are inputs: the reference's expsum_coeffs for the interval of 3 x lap(6), zeta 24
    p = T.ExpSumPreconditioner(fac, z["inv_alpha"], z["inv_beta"], T.RoundSpec(1e-12),
                               quad_bound=float(z["inv_bound"]))
    qx = T.TTVector(cores(z, "inv_qx"), device=cuda)
    got = T.precond_apply(p, qx)
    assert list(got.ranks) == list(z["inv_ranks"])
    assert _rel(_dense(got), z["inv_out"]) <= 1e-10
    # approximate inverse: ||P^{-1} A x - x|| <= 10 * quadrature bound (reference property)
    x = T.TTVector(cores(z, "inv_x"), device=cuda)
    assert T.tt_norm(T.tt_combine([got, x], [1.0, -1.0])) <= 10 * p.quad_bound + 1e-12


def test_precond_accumulation_modes_golden(cuda, z):
    fac = [_lap(5)] * 3
    spec = T.RoundSpec(1e-10, max_rank=12)
    seq = T.ExpSumPreconditioner(fac, z["acc_alpha"], z["acc_beta"], spec, accumulate="sequential")
    st = T.ExpSumPreconditioner(fac, z["acc_alpha"], z["acc_beta"], spec, accumulate="stream")
    v = T.TTVector(cores(z, "acc_v"), device=cuda)
    a, b = _dense(T.precond_apply(seq, v)), _dense(T.precond_apply(st, v))
    assert _rel(a, z["acc_seq"]) <= 1e-10
    assert _rel(b, z["acc_stream"]) <= 1e-10
    assert _rel(b, a) <= 1e-6


def test_precond_linearity(cuda):
    z = load("precond.npz")
    p = T.ExpSumPreconditioner([_lap(4)] * 2, z["acc_alpha"], z["acc_beta"], T.RoundSpec(1e-12))
    a = T.tt_random([4, 4], [2], seed=8, device=cuda)
    b = T.tt_random([4, 4], [1], seed=9, device=cuda)
    lhs = T.precond_apply(p, T.tt_combine([a, b], [2.0, -3.0]))
    rhs = T.tt_combine([T.precond_apply(p, a), T.precond_apply(p, b)], [2.0, -3.0])
    assert T.tt_norm(T.tt_combine([lhs, rhs], [1.0, -1.0])) <= 1e-6 * max(T.tt_norm(lhs), 1.0)


def _cfg(z, name):
    c = z[f"{name}_cfg"]
    return T.SolverConfig(maxit=int(c[0]), tol=float(c[1]), ell=int(c[2]), eta=float(c[3]),
                          max_rank=None if c[4] < 0 else int(c[4]), sketch_rows=int(c[5]),
                          oversampling=int(c[6]), solution_rank=None if c[7] < 0 else int(c[7]),
                          seed=int(c[8]))


def test_spgmres_identity_preconditioner_golden(cuda, z):
    """beta = 0: P^{-1} is a 1e-14 rounding; history equals the plain solver's
    (test_solvers.py:256-266) and the reference's."""
    a = T.TTOperator(cores(z, "sp_id_op"), device=cuda)
    b = T.TTVector(cores(z, "sp_id_b"), device=cuda)
    s = T.KhatriRaoSketch(factors(z, "sp_id"), device=cuda)
    def drm(prefix):
        cs = [torch.as_tensor(c, device=cuda) for c in cores(z, prefix)]
        return T.TTDRM(b.dims, [1] + [c.shape[2] for c in cs], cs)

    frame = T.StreamFrame(right=drm("sp_id_right"), left=drm("sp_id_left"))
    p = T.ExpSumPreconditioner([np.zeros((5, 5))] * 3, [1.0], [0.0], T.RoundSpec(1e-14))
    cfg = _cfg(z, "sp_id")
    x, rep = T.tt_spgmres(a, p, b, None, cfg, s, frame)
    _, rep_u = T.tt_sgmres(a, b, None, cfg, s, frame)
    assert rep.iterations == int(z["sp_id_iters"]) == rep_u.iterations
    np.testing.assert_allclose(rep.res_sketched, z["sp_id_res"], rtol=1e-6)
    np.testing.assert_allclose(rep.res_sketched, rep_u.res_sketched, rtol=1e-6)
    assert _rel(_dense(x), z["sp_id_x"]) <= 1e-7


def test_spgmres_expsum_pde_golden(cuda, z):
    """Exp-sum preconditioned convection-diffusion, d=3 n=16 zeta 17
    (test_solvers.py:268-285): identical iteration count, final residual within
    1e-8, solution within 1e-8 of the reference's."""
    a = T.TTOperator(cores(z, "sp_pde_op"), device=cuda)
    b = T.TTVector(cores(z, "sp_pde_b"), device=cuda)
    s = T.KhatriRaoSketch(factors(z, "sp_pde"), device=cuda)
    fac = [z[f"sp_pde_fac{k}"] for k in range(3)]
    p = T.ExpSumPreconditioner(fac, z["sp_pde_alpha"], z["sp_pde_beta"], T.RoundSpec(1e-9, max_rank=30))
    x, rep = T.tt_spgmres(a, p, b, None, _cfg(z, "sp_pde"), s)
    assert rep.converged and rep.iterations == int(z["sp_pde_iters"])
    np.testing.assert_allclose(rep.res_sketched, z["sp_pde_res"], rtol=1e-6, atol=1e-12)
    assert abs(rep.res_sketched[-1] - z["sp_pde_res"][-1]) <= 1e-8
    assert _rel(_dense(x), z["sp_pde_x"]) <= 1e-8
    assert T.true_residual(a, b, x) <= 1e-7
