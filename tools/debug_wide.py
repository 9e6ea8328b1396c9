"""Checks of the wide (> 160 column) QR / SVD paths through the ABI, in the
layouts the rounding drivers use (column-major Q, transposed B)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2409_09471_b200 import _lib
import oracle as O
import paper_2409_09471_b200 as T
lib = _lib.load()
dev = torch.device("cuda", 0)


def qr(A, a_col, q_col):
    m, l = A.shape
    k = min(m, l)
    if a_col:
        At = torch.as_tensor(np.ascontiguousarray(A.T), device=dev); a_rs, a_cs = 1, m
    else:
        At = torch.as_tensor(A, device=dev); a_rs, a_cs = l, 1
    if q_col:
        Qt = torch.empty((k, m), dtype=torch.float64, device=dev); q_rs, q_cs = 1, m
    else:
        Qt = torch.empty((m, k), dtype=torch.float64, device=dev); q_rs, q_cs = k, 1
    R = torch.empty((k, l), dtype=torch.float64, device=dev)
    ws = _lib.workspace(lib.ttk_qr_ws_bytes(m, l), dev)
    _lib.check(lib.ttk_qr_auto(m, l, At.data_ptr(), a_rs, a_cs, Qt.data_ptr(), q_rs, q_cs, R.data_ptr(),
                               ws.data_ptr(), ws.numel(), _lib.stream_ptr(dev)))
    Q = Qt.cpu().numpy()
    Q = Q.T if q_col else Q
    return Q, R.cpu().numpy()


rng = np.random.default_rng(0)
B = rng.standard_normal((6000, 100))
cases = {"gauss4096x200": rng.standard_normal((4096, 200)), "dup6000x200": np.concatenate([B, B], axis=1),
         "gauss64x200": rng.standard_normal((64, 200)), "zero900x161": np.zeros((900, 161)),
         "gauss2560x200": rng.standard_normal((2560, 200))}
for name, A in cases.items():
    for a_col in (False, True):
        for q_col in (False, True):
            Q, R = qr(A, a_col, q_col)
            k = Q.shape[1]
            orth = np.abs(Q.T @ Q - np.eye(k)).max()
            rec = np.linalg.norm(Q @ R - A) / max(np.linalg.norm(A), 1e-300)
            colrec = [float(np.linalg.norm((Q @ R - A)[:, c0:c0 + 67])) for c0 in range(0, A.shape[1], 67)]
            print(f"{name} a_col={a_col} q_col={q_col}: orth {orth:.2e} rec {rec:.2e} per-panel {['%.1e' % x for x in colrec]}",
                  flush=True)

from paper_2409_09471_b200 import configs
C = configs.config2()
x = T.TTVector(C["x"], device=dev)
for cap in (40, 150, 170):
    got = T.tt_round(x, T.RoundSpec(0.0, cap), zero_rel=None)
    want = O.tt_round(C["x"], 0.0, cap, zero_rel=None)
    print("config2 tt_round cap", cap, "ranks equal", list(got.ranks) == [1] + [c.shape[2] for c in want],
          "rel_diff", O.rel_diff([c.cpu().numpy() for c in got.cores], want), flush=True)
