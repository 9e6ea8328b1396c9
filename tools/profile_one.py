"""Single-kernel workloads for ncu --set full captures."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2409_09471_b200 as T
from paper_2409_09471_b200 import configs
dev = torch.device("cuda", 0)
which = sys.argv[1]
if which == "matvec":
    C = configs.config3()
    op = T.TTOperator(C["op"], device=dev); x = T.TTVector(C["x"], device=dev)
    y = T.tt_matvec(op, x)
    for _ in range(3):
        T.tt_matvec(op, x, out=y.cores)
elif which == "step":
    C = configs.config3()
    op = T.TTOperator(C["op"], device=dev); x = T.TTVector(C["x"], device=dev)
    drm = [torch.as_tensor(g, device=dev) for g in C["drm"]]
    for _ in range(2):
        T.tt_truncate_left_orth(T.rto_sweeps(T.tt_matvec(op, x), drm), T.RoundSpec(0.0, 64))
torch.cuda.synchronize()
print("ok", which)
