"""Same-process A/B of ttk_gemm_tma variants: ab/lib_<name>.so for each name,
shapes MxNxK, interleaved timing (diagnostics)."""
import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
names = sys.argv[1].split(",")
shapes = [tuple(int(v) for v in a.split("x")) for a in sys.argv[2:]]
libs = {}
for nm in names:
    L = ctypes.CDLL(os.path.join(root, "ab", f"lib_{nm}.so"))
    L.ttk_gemm_tma.argtypes = [ctypes.c_int] * 3 + [ctypes.c_double, ctypes.c_void_p, ctypes.c_longlong,
                                                    ctypes.c_void_p, ctypes.c_longlong, ctypes.c_double,
                                                    ctypes.c_void_p, ctypes.c_longlong, ctypes.c_void_p]
    libs[nm] = L
dev = torch.device("cuda", 0); st = torch.cuda.current_stream(dev)
for M, N, K in shapes:
    A = torch.randn(M, K, dtype=torch.float64, device=dev); B = torch.randn(K, N, dtype=torch.float64, device=dev)
    C = torch.empty(M, N, dtype=torch.float64, device=dev); ref = A @ B
    res = {nm: [] for nm in names}; err = {}
    for rep in range(5):
        for nm in names:
            f = lambda: libs[nm].ttk_gemm_tma(M, N, K, 1.0, A.data_ptr(), K, B.data_ptr(), N, 0.0, C.data_ptr(), N,
                                              st.cuda_stream)
            for _ in range(3): f()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            for _ in range(20): f()
            b.record(st); torch.cuda.synchronize()
            res[nm].append(a.elapsed_time(b) / 20 * 1e3)
            err[nm] = (C - ref).abs().max().item()
    fl = 2.0 * M * N * K
    print(f"{M}x{N}x{K}: " + "  ".join(f"{nm} {np.median(t):.1f} us ({fl / np.median(t) / 1e6:.1f} TF/s, err {err[nm]:.0e})"
                                        for nm, t in res.items()), flush=True)
