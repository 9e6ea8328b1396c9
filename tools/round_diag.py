"""Per-rounding GPU vs oracle error inside the config-1 solve (diagnostics).
Each tt_round the solver makes is repeated by the oracle on the same input;
the K10 difference metric is reported relative to the INPUT norm."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import oracle as O
import paper_2409_09471_b200 as T
import paper_2409_09471_b200.solvers as SV
from golden_io import cores, factors, load

cuda = torch.device("cuda", 0)
z = load("solver_cfg1.npz")
c = z["cfg1_cfg"]
cfg = T.SolverConfig(maxit=int(c[0]), tol=float(c[1]), ell=int(c[2]), eta=float(c[3]),
                     max_rank=None if c[4] < 0 else int(c[4]), sketch_rows=int(c[5]),
                     oversampling=int(c[6]), solution_rank=None if c[7] < 0 else int(c[7]),
                     seed=int(c[8]), combine_mode="stta" if c[9] else "explicit", zero_rel=None)
orig = SV.tt_round
log = []
def wrapped(v, spec, zero_rel=None):
    vin = [x.cpu().numpy() for x in v.cores]
    out = orig(v, spec, zero_rel=zero_rel)
    ref = O.tt_round(vin, spec.rel_tol, spec.max_rank, zero_rel=zero_rel)
    g = [x.cpu().numpy() for x in out.cores]
    nin = O.orth_norm(vin)
    nout = O.orth_norm(ref)
    err = O.diff_norm(g, ref)
    log.append((max(x.shape[2] for x in vin), [x.shape[2] for x in g][:-1] == [x.shape[2] for x in ref][:-1],
                err / nin, err / max(nout, 1e-300), nout / nin))
    return out
SV.tt_round = wrapped
a = T.TTOperator(cores(z, "cfg1_op"), device=cuda)
b = T.TTVector(cores(z, "cfg1_b"), device=cuda)
s = T.KhatriRaoSketch(factors(z, "cfg1"), device=cuda)
x, rep = T.tt_sgmres(a, b, None, cfg, s, T.make_solver_frame(b, cfg, seed=1))
ref = np.array(z["cfg1_res"])
print("final rel dev", abs(rep.res_sketched[-1] - ref[-1]) / ref[-1])
for i, (r, same, e_in, e_out, ratio) in enumerate(log):
    print(f"{i:3d} maxrank_in {r:4d} ranks_same {same} err/|in| {e_in:.2e} err/|out| {e_out:.2e} |out|/|in| {ratio:.2e}")
