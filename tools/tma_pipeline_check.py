"""Config-3 RTO sweeps, truncation and the fused pipeline against the oracle in a fresh
process (used to catch the TMA GEMM ordering race; diagnostics)."""
import sys, os
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import oracle as O, paper_2409_09471_b200 as T
from paper_2409_09471_b200 import configs
dev = torch.device("cuda", 0)
C = configs.config3()
spec = T.RoundSpec(C["rel_tol"], C["max_rank"])
drm = [torch.as_tensor(g, device=dev) for g in C["drm"]]
y = O.matvec(C["op"], C["x"])
Yd = T.tt_matvec(T.TTOperator(C["op"], device=dev), T.TTVector(C["x"], device=dev))
want_r = O.rto_sweeps(y, C["drm"])
got_r = T.rto_sweeps(Yd, drm)
print("rto", max(np.abs(np.abs(a.cpu().numpy())-np.abs(b)).max()/np.abs(b).max() for a,b in zip(got_r.cores, want_r)), flush=True)
want = O.truncate_left_orth(want_r, C["rel_tol"], C["max_rank"])
got_t = T.tt_truncate_left_orth(got_r, spec)
print("trunc", O.rel_diff([c.cpu().numpy() for c in got_t.cores], want), flush=True)
got = T.tt_matvec_round_rto(T.TTOperator(C["op"], device=dev), T.TTVector(C["x"], device=dev), spec, drm, device=dev)
print("pipeline", O.rel_diff([c.cpu().numpy() for c in got.cores], want), flush=True)
