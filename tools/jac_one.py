"""One l x l Jacobi SVD for ncu: python tools/jac_one.py [l] [nov]  (nov: no V, the Gram truncation path)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2409_09471_b200 import _lib
lib = _lib.load(); dev = torch.device("cuda", 0); l = int(sys.argv[1]) if len(sys.argv) > 1 else 80
g = torch.Generator().manual_seed(0)
R = torch.linalg.qr(torch.randn(10 * l, l, dtype=torch.float64, generator=g))[1].to(dev).contiguous()
U = torch.empty((l, l), dtype=torch.float64, device=dev); S = torch.empty(l, dtype=torch.float64, device=dev)
V = torch.empty((l, l), dtype=torch.float64, device=dev)
vp = None if (len(sys.argv) > 2 and sys.argv[2] == "nov") else V.data_ptr()
for _ in range(3):
    lib.ttk_svd_small(l, l, R.data_ptr(), U.data_ptr(), S.data_ptr(), vp, _lib.stream_ptr(dev))
torch.cuda.synchronize(); print("ok")
