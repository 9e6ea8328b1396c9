"""Same-process A/B of Jacobi SVD variants: load ab/lib_<name>.so for each name
and time ttk_svd_small (V accumulated and not) interleaved, rounds x reps."""
import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
names = sys.argv[1].split(",")
sizes = [int(v) for v in (sys.argv[2:] or ["80", "50"])]
libs = {}
for nm in names:
    L = ctypes.CDLL(os.path.join(root, "ab", f"lib_{nm}.so"))
    L.ttk_svd_small.argtypes = [ctypes.c_int, ctypes.c_int] + [ctypes.c_void_p] * 5
    libs[nm] = L
dev = torch.device("cuda", 0); st = torch.cuda.current_stream(dev)
for l in sizes:
    g = np.random.default_rng(l)
    R = np.linalg.qr(g.standard_normal((10 * l, l)))[1]
    Bt = torch.as_tensor(np.ascontiguousarray(R.T), device=dev)
    U = torch.empty((l, l), dtype=torch.float64, device=dev); S = torch.empty(l, dtype=torch.float64, device=dev)
    V = torch.empty((l, l), dtype=torch.float64, device=dev)
    res = {(nm, v): [] for nm in names for v in (0, 1)}
    errs = {}
    for rep in range(5):
        for nm in names:
            for v in (0, 1):
                call = lambda: libs[nm].ttk_svd_small(l, l, Bt.data_ptr(), U.data_ptr(), S.data_ptr(),
                                                      V.data_ptr() if v else None, st.cuda_stream)
                for _ in range(2): call()
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st)
                for _ in range(10): call()
                b.record(st); torch.cuda.synchronize()
                res[(nm, v)].append(a.elapsed_time(b) / 10 * 1e3)
                if rep == 0:
                    sl = np.linalg.svd(R, compute_uv=False)
                    u = U.cpu().numpy(); sv = S.cpu().numpy()
                    errs[(nm, v)] = (np.abs(sv - sl).max() / sl[0], np.abs(u.T @ u - np.eye(l)).max())
    print(f"{l}x{l}: " + "  ".join(f"{nm}{'+V' if v else ''} {np.median(t):.1f}" for (nm, v), t in res.items()),
          flush=True)
    print("   errors (S rel, U orth): " + "  ".join(f"{nm}{'+V' if v else ''} {e[0]:.1e}/{e[1]:.1e}"
                                                  for (nm, v), e in errs.items()), flush=True)
