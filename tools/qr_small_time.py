"""ttk_qr_auto timing on the solver's small shapes (diagnostics)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2409_09471_b200 import _lib
lib = _lib.load(); dev = torch.device("cuda", 0); st = _lib.stream_ptr(dev)
for (m, l) in [(5376, 21), (2560, 10), (5376, 40), (10240, 80)]:
    g = torch.Generator(device=dev); g.manual_seed(1)
    A = torch.randn((m, l), dtype=torch.float64, device=dev, generator=g)
    Q = torch.empty_like(A); R = torch.empty((l, l), dtype=torch.float64, device=dev)
    ws = _lib.workspace(lib.ttk_qr_ws_bytes(m, l) + (64 << 20), dev)
    call = lambda: _lib.check(lib.ttk_qr_auto(m, l, A.data_ptr(), l, 1, Q.data_ptr(), l, 1, R.data_ptr(), ws.data_ptr(), ws.numel(), st))
    for _ in range(3): call()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20): call()
    b.record(); torch.cuda.synchronize()
    err = float((Q @ R - A).abs().max()); orth = float((Q.T @ Q - torch.eye(l, device=dev, dtype=torch.float64)).abs().max())
    print(f"{m}x{l}: {a.elapsed_time(b) / 20 * 1e3:.1f} us  |QR-A| {err:.1e} |QtQ-I| {orth:.1e}")
