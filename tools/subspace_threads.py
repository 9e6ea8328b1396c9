"""Concurrency check: several host threads, each with its own stream and buffers,
run the subspace kernel / the blocked Cholesky back to back (diagnostics)."""
import os, sys, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2409_09471_b200 import _lib
lib = _lib.load(); dev = torch.device("cuda", 0)
which = sys.argv[1] if len(sys.argv) > 1 else "subspace"
l, r = 80, 64
rng = np.random.default_rng(0)
U, _ = np.linalg.qr(rng.standard_normal((l, l)))
sv = np.concatenate([np.linspace(1.3, 1.0, r), 1e-3 * np.linspace(1.0, 0.1, l - r)])
G0 = (U * sv**2) @ U.T
errs = []
def worker(i):
    try:
        s = torch.cuda.Stream(device=dev)
        with torch.cuda.stream(s):
            G = torch.as_tensor(G0, device=dev).clone()
            F = torch.zeros((l, l), dtype=torch.float64, device=dev); Mt = torch.zeros_like(F)
            flag = torch.zeros(1, dtype=torch.int32, device=dev); info = torch.zeros(4, dtype=torch.float64, device=dev)
            R = torch.zeros_like(F)
            for it in range(300):
                if which == "subspace":
                    _lib.check(lib.ttk_debug_trunc_subspace(l, r, G.data_ptr(), F.data_ptr(), Mt.data_ptr(), flag.data_ptr(),
                                                            info.data_ptr(), None, s.cuda_stream))
                else:
                    _lib.check(lib.ttk_debug_chol(l, G.data_ptr(), R.data_ptr(), flag.data_ptr(), s.cuda_stream))
            s.synchronize()
            print(i, "ok", int(flag.item()), info.cpu().numpy())
    except Exception as e:
        errs.append(e); print(i, "ERR", e)
ts = [threading.Thread(target=worker, args=(i,)) for i in range(4)]
[t.start() for t in ts]; [t.join() for t in ts]
torch.cuda.synchronize()
print("errors", len(errs))
