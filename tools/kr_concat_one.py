"""One Khatri-Rao sketch batch (config 4, fused kernel) and one SURVEY-8(d) axpy
concatenation (ranks [120, 60, 60, 60] -> 300, d = 50, n = 256) for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2409_09471_b200 as T
from paper_2409_09471_b200 import configs
dev = torch.device("cuda", 0)
which = sys.argv[1] if len(sys.argv) > 1 else "kr"
if which == "kr":
    C4 = configs.config4(nvec=int(os.environ.get("NVEC", "64")))
    sk = T.KhatriRaoSketch(C4["factors"], device=dev)
    vs = [T.TTVector(v, device=dev) for v in C4["vecs"]]
    for _ in range(2):
        T.kr_apply_batch(sk, vs)
else:
    rng = np.random.default_rng(0)
    d, n = 50, 256
    def tt(r):
        return T.TTVector([torch.randn((1 if k == 0 else r, n, 1 if k == d - 1 else r), dtype=torch.float64,
                                       device=dev) for k in range(d)])
    terms = [tt(120), tt(60), tt(60), tt(60)]
    for _ in range(2):
        T.tt_combine(terms, [1.0, -0.3, 0.2, -0.1])
torch.cuda.synchronize(); print("ok")
