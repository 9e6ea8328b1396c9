"""Time the standalone blocked Cholesky (the truncation's Gram path) and print
its phase clocks: python tools/chol_one.py [l] (diagnostics)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2409_09471_b200 import _lib
lib = _lib.load(); dev = torch.device("cuda", 0); st = _lib.stream_ptr(dev)
l = int(sys.argv[1]) if len(sys.argv) > 1 else 80
C = np.random.default_rng(0).standard_normal((l, 100 * l))
G = torch.as_tensor(C @ C.T, device=dev); R = torch.empty((l, l), dtype=torch.float64, device=dev)
stt = torch.zeros(1, dtype=torch.int32, device=dev)
call = lambda: lib.ttk_debug_chol(l, G.data_ptr(), R.data_ptr(), stt.data_ptr(), st)
for _ in range(3): call()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20): call()
b.record(); torch.cuda.synchronize()
prof = torch.zeros(8, dtype=torch.int64, device=dev)
lib.ttk_debug_chol_profile(prof.data_ptr()); call(); torch.cuda.synchronize(); lib.ttk_debug_chol_profile(None)
p = prof.cpu().numpy(); n = max(p[5], 1)
r = R.cpu().numpy()
print(f"{l}x{l}: {a.elapsed_time(b) / 20 * 1e3:.1f} us (status {int(stt.item())}, |R^T R - G|/|G| "
      f"{np.abs(r.T @ r - G.cpu().numpy()).max() / np.abs(G.cpu().numpy()).max():.1e}); cycles: load {p[0]/n:.0f} "
      f"diag {p[1]/n:.0f} panel {p[2]/n:.0f} trailing {p[3]/n:.0f} epilogue {p[4]/n:.0f}", flush=True)
