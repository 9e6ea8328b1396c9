"""Config-5 RTO-mode solve: GPU vs oracle solution diagnostics."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O
import paper_2409_09471_b200 as T
from paper_2409_09471_b200 import configs
dev = torch.device("cuda", 0)
C = configs.config5(0)
cfg = T.SolverConfig(**C["cfg"], zero_rel=None, rounding="rto")
a = T.TTOperator(C["op"], device=dev)
b = T.TTVector(C["b"], device=dev)
s = T.kr_sketch_new(C["dims"], cfg.sketch_rows, seed=C["sketch_seed"], device=dev)
x, rep = T.tt_sgmres(a, b, None, cfg, s, T.make_solver_frame(b, cfg, seed=C["frame_seed"]))
xg = [c.cpu().numpy() for c in x.cores]
ocfg = {"maxit": cfg.maxit, "tol": cfg.tol, "ell": cfg.ell, "eta": cfg.eta, "max_rank": cfg.max_rank,
        "oversampling": cfg.oversampling, "seed": cfg.seed, "zero_rel": None}
drm = [g.cpu().numpy() for g in T.solver_rto_drm(b.dims, cfg, device=dev).cores]
f_np = [f.cpu().numpy() for f in s.factors]
ox, orep = O.sgmres(C["op"], C["b"], ocfg, f_np, frame=O.solver_frame(C["b"], ocfg, seed=C["frame_seed"]),
                    rounding="rto", rto_drm=drm)
print("ranks gpu", [c.shape[2] for c in xg][:10], "oracle", [c.shape[2] for c in ox][:10])
print("core max gpu", ["%.1e" % np.abs(c).max() for c in xg[:6]], "oracle", ["%.1e" % np.abs(c).max() for c in ox[:6]])
print("finite", all(np.isfinite(c).all() for c in xg), all(np.isfinite(c).all() for c in ox))
print("orth_norm gpu", O.orth_norm(xg), "oracle", O.orth_norm(ox), "tt_norm gpu", T.tt_norm(x))
fp = O.kr_factors_new(C["dims"], 24, seed=777)
pg, po = O.kr_apply(fp, xg), O.kr_apply(fp, ox)
print("probe rel diff", np.linalg.norm(pg - po) / np.linalg.norm(po))
print("rel_diff", O.rel_diff(xg, ox), "reverse", O.rel_diff(ox, xg))
