"""Exp-sum preconditioner, CPU side: argument validation of the package's
setup (the coefficients are caller inputs, taken from the reference's own
expsum_coeffs output in golden/precond.npz), and the oracle's mode_multiply / exp-sum apply / preconditioned sGMRES pinned to the
reference's outputs on the cases of pkg/tests/test_precond.py and
test_solvers.py:255-285."""

import numpy as np
import pytest
import scipy.linalg

import oracle as O
import paper_2409_09471_b200 as T
from golden_io import cores, factors, load


@pytest.fixture(scope="module")
def z():
    return load("precond.npz")


def test_host_errors():
    with pytest.raises(T.ShapeMismatch):
        T.matrix_exp(np.zeros((2, 3)))
    with pytest.raises(ValueError):
        T.matrix_exp(np.array([[np.inf, 0.0], [0.0, 1.0]]))
    assert np.array_equal(T.matrix_exp(np.zeros((4, 4))), np.eye(4))
    with pytest.raises(ValueError):
        T.ExpSumPreconditioner([np.eye(2)], [1.0, 2.0], [1.0], T.RoundSpec(0.0))
    with pytest.raises(ValueError):
        T.ExpSumPreconditioner([np.eye(2)], [1.0], [-1.0], T.RoundSpec(0.0))
    with pytest.raises(ValueError):
        T.ExpSumPreconditioner([np.eye(2)], [1.0], [1.0], T.RoundSpec(0.0), accumulate="bogus")


def _exps(factors_, beta):
    return [[scipy.linalg.expm(-b * f) for f in factors_] for b in beta]


def _lap(n):
    return -(-2.0 * np.eye(n) + np.diag(np.ones(n - 1), 1) + np.diag(np.ones(n - 1), -1))


def _rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b)


def test_oracle_mode_multiply_golden(z):
    mats = [z[f"mm_mat{k}"] for k in range(3)]
    got = O.mode_multiply(cores(z, "mm_in"), mats)
    for g, w in zip(got, cores(z, "mm_out")):
        assert g.shape == w.shape
        assert np.abs(g - w).max() <= 1e-14 * np.abs(w).max()


def test_oracle_expsum_apply_golden(z):
    fac = [_lap(6)] * 3
    out = O.expsum_apply(cores(z, "inv_qx"), _exps(fac, z["inv_beta"]), z["inv_alpha"], 1e-12)
    assert [1] + [c.shape[2] for c in out] == list(z["inv_ranks"])
    assert _rel(O.to_dense(out), z["inv_out"]) <= 1e-10
    fac = [_lap(5)] * 3
    v = cores(z, "acc_v")
    exps = _exps(fac, z["acc_beta"])
    seq = O.expsum_apply(v, exps, z["acc_alpha"], 1e-10, 12)
    assert _rel(O.to_dense(seq), z["acc_seq"]) <= 1e-10
    # stream mode: frame at the rank cap, stream_seed 0 (precond.py:272-278)
    st = O.expsum_apply(v, exps, z["acc_alpha"], 1e-10, 12, accumulate="stream",
                        frame=O.frame_new([5, 5, 5], [12, 12], 20, 0))
    assert _rel(O.to_dense(st), z["acc_stream"]) <= 1e-10


def _ocfg(z, name):
    c = z[f"{name}_cfg"]
    return {"maxit": int(c[0]), "tol": float(c[1]), "ell": int(c[2]), "eta": float(c[3]),
            "max_rank": None if c[4] < 0 else int(c[4]), "oversampling": int(c[6]),
            "solution_rank": None if c[7] < 0 else int(c[7]), "seed": int(c[8])}


@pytest.mark.parametrize("name", ["sp_id", "sp_pde"])
def test_oracle_spgmres_golden(z, name):
    spec = z[f"{name}_spec"]
    rel, cap = float(spec[0]), None if spec[1] < 0 else int(spec[1])
    b = cores(z, f"{name}_b")
    n = b[0].shape[1]
    if name == "sp_id":
        exps = [[np.eye(n)] * 3]
        frame = (cores(z, f"{name}_left"), cores(z, f"{name}_right"))
    else:
        exps = _exps([z[f"sp_pde_fac{k}"] for k in range(3)], z[f"{name}_beta"])
        frame = None
    alpha = z[f"{name}_alpha"]
    ocfg = _ocfg(z, name)
    x, rep = O.sgmres(cores(z, f"{name}_op"), b, ocfg, factors(z, name), frame=frame,
                      precond=lambda v: O.expsum_apply(v, exps, alpha, rel, cap))
    assert rep["iterations"] == int(z[f"{name}_iters"])
    assert rep["converged"] == bool(z[f"{name}_conv"])
    np.testing.assert_allclose(rep["res_sketched"], z[f"{name}_res"], rtol=1e-6, atol=1e-12)
    assert _rel(O.to_dense(x), z[f"{name}_x"]) <= 1e-8
