"""Config-5 final recovery (stream_recover) on the GPU vs the oracle on the same sketch pair."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as O
import paper_2409_09471_b200 as T
from paper_2409_09471_b200 import configs, streaming, solvers, _lib
dev = torch.device("cuda", 0)
C = configs.config5(0)
cfg = T.SolverConfig(**C["cfg"], zero_rel=None)
a = T.TTOperator(C["op"], device=dev)
b = T.TTVector(C["b"], device=dev)
s = T.kr_sketch_new(C["dims"], cfg.sketch_rows, seed=C["sketch_seed"], device=dev)
cap = {}
orig = solvers.stream_recover


def spy(pair, spec, zero_rel=None):
    cap["pair"], cap["spec"] = pair, spec
    return orig(pair, spec, zero_rel=zero_rel)


solvers.stream_recover = spy
x, rep = T.tt_sgmres(a, b, None, cfg, s, T.make_solver_frame(b, cfg, seed=C["frame_seed"]))
pair, spec = cap["pair"], cap["spec"]
psi = [p.cpu().numpy() for p in pair.psi]
om = [o.cpu().numpy() for o in pair.omega]
dims = list(pair.dims)
print("spec", spec.rel_tol, spec.max_rank, "x ranks", list(x.ranks)[:8], "norm", T.tt_norm(x))
# unrounded recovery: GPU vs oracle
lib = _lib.load()
d = len(psi)
lr = [1] + [o.shape[0] for o in om] + [1]
rr = [1] + [o.shape[1] for o in om] + [1]
di, li, ri = _lib.int_array(dims), _lib.int_array(lr), _lib.int_array(rr)
capn = [max(lr[mu], rr[mu]) * dims[mu] * rr[mu + 1] for mu in range(d)]
outs = [torch.empty(max(c, 1), dtype=torch.float64, device=dev) for c in capn]
out_ranks = (_lib.ctypes.c_int * (d + 1))()
is_zero = _lib.ctypes.c_int(0)
ws = _lib.workspace(lib.ttk_stream_recover_ws_bytes(d, di, li, ri), dev)
_lib.check(lib.ttk_stream_recover_cores(d, di, li, ri, _lib.ptr_array(pair.psi), _lib.ptr_array(pair.omega),
                                        streaming.PINV_RCOND, _lib.ptr_array(outs), out_ranks,
                                        _lib.ctypes.byref(is_zero), ws.data_ptr(), ws.numel(), _lib.stream_ptr(dev)))
r = list(out_ranks)
gcores = [outs[k][: r[k] * dims[k] * r[k + 1]].view(r[k], dims[k], r[k + 1]).cpu().numpy() for k in range(d)]
# oracle unrounded
lh, rh = [], []
for o in om:
    u, sv, vt = np.linalg.svd(o, full_matrices=False)
    keep = sv > 1e-12 * sv[0]
    u, sv, vt = u[:, keep], sv[keep], vt[keep]
    sq = 1.0 / np.sqrt(sv)
    lh.append(sq[:, None] * u.T)
    rh.append(vt.T * sq[None, :])
ocores = []
for mu in range(d):
    p = psi[mu]
    blk = p.reshape(p.shape[0] // dims[mu], dims[mu], p.shape[1])
    if mu > 0:
        blk = np.tensordot(lh[mu - 1], blk, axes=([1], [0]))
    if mu < d - 1:
        blk = np.tensordot(blk, rh[mu], axes=([2], [0]))
    ocores.append(blk)
print("unrounded ranks gpu", r[:8], "oracle", [1] + [c.shape[2] for c in ocores][:7])
print("omega kept gpu? sv counts", [int(np.sum(np.linalg.svd(o, compute_uv=False) > 1e-12 * np.linalg.svd(o, compute_uv=False)[0])) for o in om[:5]])
print("unrounded orth_norm gpu", O.orth_norm(gcores), "oracle", O.orth_norm(ocores))
if [c.shape for c in gcores] == [c.shape for c in ocores]:
    print("unrounded rel_diff", O.rel_diff(gcores, ocores))
# rounding: GPU tt_round of oracle cores vs oracle tt_round
gx = T.tt_round(T.TTVector(ocores, device=dev), spec, zero_rel=None)
ox = O.tt_round(ocores, spec.rel_tol, spec.max_rank, zero_rel=None)
print("round ranks gpu", list(gx.ranks)[:8], "oracle", [1] + [c.shape[2] for c in ox][:7])
print("round norms gpu", T.tt_norm(gx), "oracle", O.orth_norm(ox))
print("round rel_diff", O.rel_diff([c.cpu().numpy() for c in gx.cores], ox))
print("omega max abs per mode", ["%.1e" % np.abs(o).max() for o in om[::7]])
print("psi max abs per mode", ["%.1e" % np.abs(p).max() for p in psi[::7]])
S0 = [np.linalg.svd(o, compute_uv=False) for o in om[:3]]
from paper_2409_09471_b200 import _lib as L
def svd_gpu(B):
    k, l = B.shape
    kn = min(k, l)
    Bt = torch.as_tensor(np.ascontiguousarray(B), device=dev)
    U = torch.empty((k, kn), dtype=torch.float64, device=dev)
    S = torch.empty(kn, dtype=torch.float64, device=dev)
    V = torch.empty((l, kn), dtype=torch.float64, device=dev)
    L.check(lib.ttk_svd_small(k, l, Bt.data_ptr(), U.data_ptr(), S.data_ptr(), V.data_ptr(), L.stream_ptr(dev)))
    return S.cpu().numpy()
for i in range(3):
    sg = svd_gpu(om[i])
    print("mode", i + 1, "lapack", ["%.2e" % x for x in S0[i][:8]], "gpu", ["%.2e" % x for x in sg[:8]])
