"""Concurrency check of the TMA GEMM: host threads on their own streams run
ttk_gemm_tma_strided on their own buffers (inputs and references made before the
threads start); lock=1 serialises the host calls only (diagnostics)."""
import os, sys, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2409_09471_b200 import _lib
lib = _lib.load(); dev = torch.device("cuda", 0)
nthr = int(sys.argv[1]) if len(sys.argv) > 1 else 2
use_lock = len(sys.argv) > 2 and sys.argv[2] == "1"
shapes = [(24576, 80, 192), (80, 24576, 192), (80, 10240, 192), (8192, 64, 80), (80, 80, 8192)]
data = []
for i in range(nthr):
    g = torch.Generator(device=dev); g.manual_seed(i)
    ws = torch.empty(32 << 20, dtype=torch.uint8, device=dev)
    sets = []
    for (M, N, K) in shapes:
        A = torch.randn((M, K), dtype=torch.float64, device=dev, generator=g)
        B = torch.randn((K, N), dtype=torch.float64, device=dev, generator=g)
        sets.append((M, N, K, A, B, torch.zeros((M, N), dtype=torch.float64, device=dev), A @ B))
    data.append((ws, sets, torch.cuda.Stream(dev)))
torch.cuda.synchronize()
lock = threading.Lock()
def worker(i):
    torch.cuda.set_device(dev)
    ws, sets, s = data[i]
    for rep in range(50):
        for (M, N, K, A, B, C, ref) in sets:
            if use_lock: lock.acquire()
            st = lib.ttk_gemm_tma_strided(M, N, K, 1.0, A.data_ptr(), K, 1, B.data_ptr(), N, 1, 0.0, C.data_ptr(), N, 1,
                                          ws.data_ptr(), ws.numel(), s.cuda_stream)
            if use_lock: lock.release()
            _lib.check(st)
ths = [threading.Thread(target=worker, args=(i,)) for i in range(nthr)]
[t.start() for t in ths]; [t.join() for t in ths]
torch.cuda.synchronize()
for i in range(nthr):
    print(i, "max |C - AB|", [float((C - ref).abs().max()) for (M, N, K, A, B, C, ref) in data[i][1]])
