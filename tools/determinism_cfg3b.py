"""The full-size config-3 test's call sequence (device call, CPU oracle, host-pipeline
call) with the differing cores printed (diagnostics)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O
import paper_2409_09471_b200 as T
from paper_2409_09471_b200 import configs
dev = torch.device("cuda", 0)
C = configs.config3()
spec = T.RoundSpec(C["rel_tol"], C["max_rank"])
drm = [torch.as_tensor(g, device=dev) for g in C["drm"]]
got = T.tt_matvec_round_rto(T.TTOperator(C["op"], device=dev), T.TTVector(C["x"], device=dev), spec, drm, device=dev)
if len(sys.argv) > 1 and sys.argv[1] == "oracle":
    y = O.matvec(C["op"], C["x"]); want = O.rto_round(y, C["drm"], C["rel_tol"], C["max_rank"])
else:
    time.sleep(float(sys.argv[1]) if len(sys.argv) > 1 else 0.0)
host = T.tt_matvec_round_rto(T.TTOperator([torch.as_tensor(g).pin_memory() for g in C["op"]]),
                             T.TTVector([torch.as_tensor(c).pin_memory() for c in C["x"]]), spec, drm, device=dev)
diff = [k for k, (a, b) in enumerate(zip(host.cores, got.cores)) if not torch.equal(a.cpu(), b.cpu())]
d2 = T.tt_add(T.TTVector([c.to(dev) for c in host.cores]), T.tt_scale(got, -1.0))
print("differing cores", diff[:6], len(diff), "tensor rel diff", float(T.tt_norm(d2)) / float(T.tt_norm(got)))
