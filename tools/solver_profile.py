"""Config-5 solve (RHS 0, RTO rounding): warm-up, then one timed solve with
phase totals; run plain and under an ncu launch list to compare the summed
kernel time with the wall time (diagnostics)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes
import torch
import paper_2409_09471_b200 as T
from paper_2409_09471_b200 import configs
dev = torch.device("cuda", 0)
j = int(sys.argv[1]) if len(sys.argv) > 1 else 0
maxit = int(sys.argv[2]) if len(sys.argv) > 2 else 60
C = configs.config5(j)
def solve(mx):
    cfg = T.SolverConfig(**{**C["cfg"], "maxit": mx}, zero_rel=None, rounding="rto")
    a = T.TTOperator(C["op"], device=dev); b = T.TTVector(C["b"], device=dev)
    s = T.kr_sketch_new(C["dims"], cfg.sketch_rows, seed=C["sketch_seed"], device=dev)
    frame = T.make_solver_frame(b, cfg, seed=C["frame_seed"])
    torch.cuda.synchronize(); t0 = time.perf_counter()
    _, rep = T.tt_sgmres(a, b, None, cfg, s, frame)
    torch.cuda.synchronize()
    return time.perf_counter() - t0, rep
solve(3)
from paper_2409_09471_b200 import _lib
lib = _lib.load()
hp0 = (ctypes.c_longlong * 2)(); lib.ttk_debug_host_profile(hp0)
n0 = lib.ttk_launch_count()
wall, rep = solve(maxit)
hp1 = (ctypes.c_longlong * 2)(); lib.ttk_debug_host_profile(hp1)
n1 = lib.ttk_launch_count()
print(json.dumps({"launches": n1 - n0, "host_syncs": hp1[0] - hp0[0], "sync_wait_s": (hp1[1] - hp0[1]) * 1e-9}))
print(json.dumps({"wall_s": wall, "iterations": rep.iterations, "it_per_s": rep.iterations / wall,
                  "phase_s": rep.phase_totals(), "ranks": rep.basis_rank}))
