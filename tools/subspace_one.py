"""Time the gap-certified subspace kernel of the truncation on real config-3
Grams (the unfoldings of the RTO output, last cores) and print its phase
clocks: python tools/subspace_one.py [ncores] (diagnostics)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2409_09471_b200 as T
from paper_2409_09471_b200 import _lib, configs
lib = _lib.load(); dev = torch.device("cuda", 0); st = _lib.stream_ptr(dev)
ncores = int(sys.argv[1]) if len(sys.argv) > 1 else 3
C = configs.config3()
y = T.tt_matvec(T.TTOperator(C["op"], device=dev), T.TTVector(C["x"], device=dev))
lo = T.rto_sweeps(y, [torch.as_tensor(g, device=dev) for g in C["drm"]])
r = 64
cur = lo.cores[-1]
for k in range(len(lo.cores) - 1, len(lo.cores) - 1 - ncores, -1):
    r0 = cur.shape[0]
    Cm = cur.reshape(r0, -1)
    G = (Cm @ Cm.T).contiguous()
    l = r0
    F = torch.zeros((l, l), dtype=torch.float64, device=dev); Mt = torch.zeros_like(F)
    flag = torch.zeros(1, dtype=torch.int32, device=dev); info = torch.zeros(4, dtype=torch.float64, device=dev)
    call = lambda prof=None: lib.ttk_debug_trunc_subspace(l, r, G.data_ptr(), F.data_ptr(), Mt.data_ptr(),
                                                          flag.data_ptr(), info.data_ptr(), prof, st)
    for _ in range(3): call()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20): call()
    b.record(); torch.cuda.synchronize()
    prof = torch.zeros(12, dtype=torch.int64, device=dev)
    call(prof.data_ptr()); torch.cuda.synchronize()
    p = prof.cpu().numpy(); i = info.cpu().numpy()
    ev = np.linalg.eigvalsh(G.cpu().numpy())[::-1]
    sv = np.sqrt(np.maximum(ev, 0))
    print(f"core {k}: l={l} r={r}: {a.elapsed_time(b) / 20 * 1e3:.1f} us flag {int(flag.item())} bound {i[0]:.1e} "
          f"tau/lmin {i[1]:.1e} iters {int(i[2])} max|MF-I| {i[3]:.1e}; s1/sr {sv[0]/sv[r-1]:.1f} sr/sr+1 {sv[r-1]/sv[r]:.1f}; cycles: "
          f"load {p[0]} init-products {p[1]} chol+inv {p[2]} iter-products {p[3]} out {p[4]}; chol: diag {p[5]} panel {p[6]} trailing {p[7]} inverse {p[8]}", flush=True)
    Y = Mt[:, :r].T @ Cm
    print(f"   |Y Y^T - I| {float((Y @ Y.T - torch.eye(r, device=dev, dtype=torch.float64)).abs().max()):.1e}", flush=True)
    # next core's unfolding: C_{k-1} x_3 F  (F = C Y^T, l x r)
    prev = lo.cores[k - 1]
    cur = (prev.reshape(-1, l) @ F[:, :r]).reshape(prev.shape[0], prev.shape[1], r)
