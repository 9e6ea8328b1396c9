"""Roundoff sensitivity of the small reference solver cases (golden
solver_small.npz) in the CPU oracle: inject 1e-16 relative noise into every
rounded TT and report how far the final sketched residual moves -- the floor
below which no backward-stable implementation (the reference's LAPACK or the
B200 kernels) can reproduce another's final residual."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import oracle as O
import oracle.ttoracle as OT
from golden_io import cores, factors, load

z = load("solver_small.npz")
rng = np.random.default_rng(0)
orig = OT.tt_round


def noisy(v, rel, cap, zero_rel=None):
    out = orig(v, rel, cap, zero_rel=zero_rel)
    return [c * (1.0 + 1e-16 * rng.standard_normal(c.shape)) for c in out]


for name in z["sv_names"]:
    c = z[f"{name}_cfg"]
    cfg = {"maxit": int(c[0]), "tol": float(c[1]), "ell": int(c[2]), "eta": float(c[3]),
           "max_rank": None if c[4] < 0 else int(c[4]), "oversampling": int(c[6]),
           "solution_rank": None if c[7] < 0 else int(c[7]), "seed": int(c[8]),
           "combine_mode": "stta" if c[9] else "explicit"}
    ref = np.array(z[f"{name}_res"])
    OT.tt_round = noisy
    for trial in range(3):
        _, rep = O.sgmres(cores(z, f"{name}_op"), cores(z, f"{name}_b"), cfg, factors(z, name))
        h = np.array(rep["res_sketched"])
        n = min(len(h), len(ref))
        d = np.abs(h[:n] - ref[:n])
        print(f"{name} trial {trial}: iters {rep['iterations']} (ref {len(ref)}) final {h[-1]:.6e} "
              f"|d_final| {abs(h[-1] - ref[-1]):.2e} rel {abs(h[-1] - ref[-1]) / ref[-1]:.2e} "
              f"max rel {np.max(d / ref[:n]):.2e}")
    OT.tt_round = orig
