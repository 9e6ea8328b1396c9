"""Fused CholeskyQR2 under concurrency: host threads / one thread with several
streams, each with its own buffers; checks |QR - A| and |Q^T Q - I| (diagnostics)."""
import os, sys, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2409_09471_b200 import _lib
lib = _lib.load(); dev = torch.device("cuda", 0)
nthr = int(sys.argv[1]) if len(sys.argv) > 1 else 2
mode = sys.argv[2] if len(sys.argv) > 2 else "threads"
m, l = 10240, 80
data = []
for i in range(nthr):
    g = torch.Generator(device=dev); g.manual_seed(i)
    A = torch.randn((m, l), dtype=torch.float64, device=dev, generator=g)
    data.append((A, torch.zeros_like(A), torch.zeros((l, l), dtype=torch.float64, device=dev),
                 torch.empty(lib.ttk_qr_ws_bytes(m, l) + (64 << 20), dtype=torch.uint8, device=dev), torch.cuda.Stream(dev)))
torch.cuda.synchronize()
worst = [[0.0, 0.0] for _ in range(nthr)]
def one(i):
    A, Q, R, ws, s = data[i]
    _lib.check(lib.ttk_qr_auto(m, l, A.data_ptr(), l, 1, Q.data_ptr(), l, 1, R.data_ptr(), ws.data_ptr(), ws.numel(), s.cuda_stream))
def check(i):
    A, Q, R, ws, s = data[i]
    worst[i][0] = max(worst[i][0], float((Q @ R - A).abs().max()))
    worst[i][1] = max(worst[i][1], float((Q.T @ Q - torch.eye(l, device=dev, dtype=torch.float64)).abs().max()))
def worker(i):
    torch.cuda.set_device(dev)
    with torch.cuda.stream(data[i][4]):
        for rep in range(30):
            for _ in range(5): one(i)
            data[i][4].synchronize(); check(i)
if mode == "threads":
    ths = [threading.Thread(target=worker, args=(i,)) for i in range(nthr)]
    [t.start() for t in ths]; [t.join() for t in ths]
else:
    for rep in range(30):
        for _ in range(5):
            for i in range(nthr): one(i)
        torch.cuda.synchronize()
        for i in range(nthr): check(i)
torch.cuda.synchronize()
print(mode, worst)
