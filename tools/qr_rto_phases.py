"""Phase timestamps (globaltimer) of the fused CholeskyQR2 as called by the
config-3 RTO left sweep (the last call of the sweep), diagnostics."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2409_09471_b200 as T
from paper_2409_09471_b200 import configs, _lib
lib = _lib.load(); dev = torch.device("cuda", 0)
C = configs.config3()
drm = [torch.as_tensor(g, device=dev) for g in C["drm"]]
y = T.tt_matvec(T.TTOperator(C["op"], device=dev), T.TTVector(C["x"], device=dev))
T.rto_sweeps(y, drm); torch.cuda.synchronize()
names = ["load+gram1", "reduce1", "chol1", "trsm+gram2", "reduce2", "nearid", "Q"]
for rep in range(3):
    ts = torch.zeros(16, dtype=torch.int64, device=dev)
    lib.ttk_debug_fused_qr_profile(ts.data_ptr())
    T.rto_sweeps(y, drm); torch.cuda.synchronize()
    lib.ttk_debug_fused_qr_profile(None)
    t = ts.cpu().numpy(); idx = [0, 1, 2, 3, 4, 5, 6, 15]
    print({names[i]: round((t[idx[i + 1]] - t[idx[i]]) / 1e3, 2) for i in range(7)}, "total_us", (t[15] - t[0]) / 1e3,
          flush=True)
