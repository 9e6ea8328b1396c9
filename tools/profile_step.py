"""One warm-up + N profiled steps of a workload (for ncu launch lists)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2409_09471_b200 as T
from paper_2409_09471_b200 import configs

which = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
dev = torch.device("cuda", 0)
if which == "cfg3":
    C = configs.config3()
    op = T.TTOperator(C["op"], device=dev)
    x = T.TTVector(C["x"], device=dev)
    drm = [torch.as_tensor(g, device=dev) for g in C["drm"]]
    spec = T.RoundSpec(0.0, 64)
    def step():
        y = T.tt_matvec(op, x)
        return T.tt_truncate_left_orth(T.rto_sweeps(y, drm), spec)
elif which == "cfg2":
    C = configs.config2()
    x = T.TTVector(C["x"], device=dev)
    drm = [torch.as_tensor(g, device=dev) for g in C["drm"]]
    def step():
        return T.tt_truncate_left_orth(T.rto_sweeps(x, drm), T.RoundSpec(0.0, 40))
if which == "cfg5":
    C = configs.config5(0)
    cfg = T.SolverConfig(**{**C["cfg"], "maxit": int(os.environ.get("MAXIT", "6"))}, zero_rel=None, rounding="rto")
    a = T.TTOperator(C["op"], device=dev); b = T.TTVector(C["b"], device=dev)
    sk = T.kr_sketch_new(C["dims"], cfg.sketch_rows, seed=C["sketch_seed"], device=dev)
    frame = T.make_solver_frame(b, cfg, seed=C["frame_seed"])
    def step():
        _, rep = T.tt_sgmres(a, b, None, cfg, sk, frame)
        print({k: round(v, 4) for k, v in rep.phase_totals().items()}, rep.basis_rank)
step()
torch.cuda.synchronize()
from paper_2409_09471_b200 import _lib
n0 = _lib.load().ttk_launch_count()
for _ in range(steps):
    step()
torch.cuda.synchronize()
print("launches per step", (_lib.load().ttk_launch_count() - n0) // steps)
