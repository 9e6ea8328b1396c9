"""TMA GEMM under host threads with pointers that change from call to call (a
ring of preallocated buffers, no allocator involvement) (diagnostics)."""
import os, sys, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2409_09471_b200 import _lib
lib = _lib.load(); dev = torch.device("cuda", 0)
nthr = int(sys.argv[1]) if len(sys.argv) > 1 else 2
mode = sys.argv[2] if len(sys.argv) > 2 else "threads"
shapes = [(24576, 80, 192), (80, 24576, 192), (80, 10240, 192), (8192, 64, 80)]
R = 6
data = []
for i in range(nthr):
    g = torch.Generator(device=dev); g.manual_seed(i)
    ws = torch.empty(32 << 20, dtype=torch.uint8, device=dev)
    sets = []
    for (M, N, K) in shapes:
        for r in range(R):
            A = torch.randn((M, K), dtype=torch.float64, device=dev, generator=g)
            B = torch.randn((K, N), dtype=torch.float64, device=dev, generator=g)
            sets.append((M, N, K, A, B, torch.zeros((M, N), dtype=torch.float64, device=dev), A @ B))
    data.append((ws, sets, torch.cuda.Stream(dev)))
torch.cuda.synchronize()
def worker(i):
    torch.cuda.set_device(dev)
    ws, sets, s = data[i]
    for rep in range(10):
        for (M, N, K, A, B, C, ref) in sets:
            _lib.check(lib.ttk_gemm_tma_strided(M, N, K, 1.0, A.data_ptr(), K, 1, B.data_ptr(), N, 1, 0.0, C.data_ptr(), N, 1,
                                                ws.data_ptr(), ws.numel(), s.cuda_stream))
if mode == "threads":
    ths = [threading.Thread(target=worker, args=(i,)) for i in range(nthr)]
    [t.start() for t in ths]; [t.join() for t in ths]
else:  # one host thread, streams interleaved
    for rep in range(10):
        for j in range(len(data[0][1])):
            for i in range(nthr):
                ws, sets, s = data[i]
                M, N, K, A, B, C, ref = sets[j]
                _lib.check(lib.ttk_gemm_tma_strided(M, N, K, 1.0, A.data_ptr(), K, 1, B.data_ptr(), N, 1, 0.0, C.data_ptr(), N, 1,
                                                    ws.data_ptr(), ws.numel(), s.cuda_stream))
torch.cuda.synchronize()
for i in range(nthr):
    print(i, "max |C - AB|", max(float((C - ref).abs().max()) for (M, N, K, A, B, C, ref) in data[i][1]))
