"""Time the truncation's 80x80 Jacobi SVD with and without V accumulation and
print the per-round phase clocks of the PROF instance (cycles per round:
rotate+apply, in-CTA move, block move, dots+reduction), diagnostics."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2409_09471_b200 import _lib
lib = _lib.load(); dev = torch.device("cuda", 0); st = torch.cuda.current_stream(dev)
l = int(sys.argv[1]) if len(sys.argv) > 1 else 80
g = np.random.default_rng(l)
R = np.linalg.qr(g.standard_normal((10 * l, l)))[1]
Bt = torch.as_tensor(np.ascontiguousarray(R.T), device=dev)
U = torch.empty((l, l), dtype=torch.float64, device=dev); S = torch.empty(l, dtype=torch.float64, device=dev)
V = torch.empty((l, l), dtype=torch.float64, device=dev)
sw = torch.zeros(1, dtype=torch.int32, device=dev)
for name, vp in (("with V", V.data_ptr()), ("no V", None)):
    call = lambda: lib.ttk_svd_small(l, l, Bt.data_ptr(), U.data_ptr(), S.data_ptr(), vp, st.cuda_stream)
    lib.ttk_debug_svd_sweeps(sw.data_ptr()); _lib.check(call()); torch.cuda.synchronize(); lib.ttk_debug_svd_sweeps(None)
    for _ in range(3): call()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(20): call()
    b.record(st); torch.cuda.synchronize()
    acc = torch.zeros(5 * 16, dtype=torch.int64, device=dev)
    lib.ttk_debug_jacobi_profile(acc.data_ptr()); _lib.check(call()); torch.cuda.synchronize(); lib.ttk_debug_jacobi_profile(None)
    p = acc.view(16, 5).cpu().numpy()
    rounds = max(int(p[0, 4]), 1)
    print(f"{l}x{l} {name}: {a.elapsed_time(b) / 20 * 1e3:.1f} us, sweeps {int(sw.item())}; cycles/round (CTA 0): "
          f"rotate {p[0,0]/rounds:.0f} move {p[0,1]/rounds:.0f} block {p[0,2]/rounds:.0f} dots {p[0,3]/rounds:.0f}",
          flush=True)
