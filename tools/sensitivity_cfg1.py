"""Roundoff sensitivity of the config-1 solve in the CPU oracle: perturb the
right-hand side by a relative 1e-15 and compare residual histories."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import oracle as O
from golden_io import cores, factors, load

z = load("solver_cfg1.npz")
c = z["cfg1_cfg"]
ocfg = {"maxit": int(c[0]), "tol": float(c[1]), "ell": int(c[2]), "eta": float(c[3]),
        "max_rank": None if c[4] < 0 else int(c[4]), "oversampling": int(c[6]), "seed": int(c[8]),
        "zero_rel": None}
a, b, f = cores(z, "cfg1_op"), cores(z, "cfg1_b"), factors(z, "cfg1")
ref = np.array(z["cfg1_res"])
rng = np.random.default_rng(0)
for trial in range(3):
    bp = [x.copy() for x in b]
    bp[-1] = bp[-1] * (1.0 + 1e-15 * rng.standard_normal(bp[-1].shape))
    _, rep = O.sgmres(a, bp, ocfg, f, frame=O.solver_frame(bp, ocfg, seed=1))
    h = np.array(rep["res_sketched"])
    d = np.abs(h - ref)
    print(f"trial {trial}: iters {rep['iterations']} final {h[-1]:.6e} |d_final| {d[-1]:.2e} "
          f"rel {d[-1]/ref[-1]:.2e} max|d| {d.max():.2e} max rel {np.max(d/ref):.2e}")

# roundoff-sized noise (1e-16 relative) injected into every rounded TT
orig = O.tt_round
def noisy(v, rel, cap, zero_rel=None):
    out = orig(v, rel, cap, zero_rel=zero_rel)
    return [c * (1.0 + 1e-16 * rng.standard_normal(c.shape)) for c in out]
O.tt_round = noisy
import oracle.ttoracle as OT
OT.tt_round = noisy
for trial in range(3):
    _, rep = O.sgmres(a, b, ocfg, f, frame=O.solver_frame(b, ocfg, seed=1))
    h = np.array(rep["res_sketched"])
    d = np.abs(h - ref)
    print(f"noisy rounding {trial}: iters {rep['iterations']} ranks_equal {rep['basis_rank'] == list(z['cfg1_ranks'])} "
          f"|d_final| {d[-1]:.2e} rel {d[-1]/ref[-1]:.2e} max rel {np.max(d/ref):.2e}")
