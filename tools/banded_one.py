"""One structured matvec of config 3 (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2409_09471_b200 as T
from paper_2409_09471_b200 import configs
dev = torch.device("cuda", 0)
C3 = configs.config3()
op, x = T.TTOperator(C3["op"], device=dev), T.TTVector(C3["x"], device=dev)
op.band_tables()
for _ in range(3):
    T.tt_matvec(op, x, structured=True)
torch.cuda.synchronize()
