"""Bit-reproducibility of the config-3 step: device-resident and host-pipeline
calls repeated in one process (diagnostics)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2409_09471_b200 as T
from paper_2409_09471_b200 import configs
dev = torch.device("cuda", 0)
C = configs.config3()
spec = T.RoundSpec(C["rel_tol"], C["max_rank"])
drm = [torch.as_tensor(g, device=dev) for g in C["drm"]]
opd = T.TTOperator(C["op"], device=dev); xd = T.TTVector(C["x"], device=dev)
oph = T.TTOperator([torch.as_tensor(g).pin_memory() for g in C["op"]])
xh = T.TTVector([torch.as_tensor(c).pin_memory() for c in C["x"]])
res = []
for i in range(4):
    res.append(("dev", T.tt_matvec_round_rto(opd, xd, spec, drm, device=dev)))
    res.append(("host", T.tt_matvec_round_rto(oph, xh, spec, drm, device=dev)))
    y = T.tt_matvec(opd, xd); lo = T.rto_sweeps(y, drm); res.append(("seq", T.tt_truncate_left_orth(lo, spec)))
    res.append(("lo", lo))
torch.cuda.synchronize()
ref = {k: v for k, v in res[:4]}
for k, v in res:
    first = [j for j, (a, b) in enumerate(zip(v.cores, ref[k].cores)) if not torch.equal(a.cpu(), b.cpu())]
    cross = [j for j, (a, b) in enumerate(zip(v.cores, ref["dev"].cores)) if not torch.equal(a.cpu(), b.cpu())] if k != "lo" else []
    print(k, "differs from first", first[:4], "| from dev", cross[:4])
