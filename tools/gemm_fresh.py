"""TMA GEMM whose operands are rewritten by a kernel on the same stream right
before every launch (fresh data in fixed buffers), several streams interleaved by
one host thread; each result is checked on the stream (diagnostics)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2409_09471_b200 import _lib
lib = _lib.load(); dev = torch.device("cuda", 0)
ns = int(sys.argv[1]) if len(sys.argv) > 1 else 3
M, N, K = (int(v) for v in sys.argv[2:5]) if len(sys.argv) > 4 else (80, 10240, 192)
R = 6
S = [torch.cuda.Stream(dev) for _ in range(ns)]
st = []
for i in range(ns):
    g = torch.Generator(device=dev); g.manual_seed(i)
    As = [torch.randn((M, K), dtype=torch.float64, device=dev, generator=g) for _ in range(R)]
    Bs = [torch.randn((K, N), dtype=torch.float64, device=dev, generator=g) for _ in range(R)]
    refs = [a @ b for a, b in zip(As, Bs)]
    st.append((As, Bs, refs, torch.zeros((M, K), dtype=torch.float64, device=dev), torch.zeros((K, N), dtype=torch.float64, device=dev),
               torch.zeros((M, N), dtype=torch.float64, device=dev), torch.zeros((), dtype=torch.float64, device=dev)))
torch.cuda.synchronize()
for rep in range(50):
    for r in range(R):
        for i, s in enumerate(S):
            As, Bs, refs, A, B, C, err = st[i]
            with torch.cuda.stream(s):
                A.copy_(As[r]); B.copy_(Bs[r])
                _lib.check(lib.ttk_gemm_tma_strided(M, N, K, 1.0, A.data_ptr(), K, 1, B.data_ptr(), N, 1, 0.0, C.data_ptr(), N, 1,
                                                    None, 0, s.cuda_stream))
                torch.maximum(err, (C - refs[r]).abs().max(), out=err)
torch.cuda.synchronize()
print("streams", ns, (M, N, K), "max errors", [float(x[6]) for x in st])
