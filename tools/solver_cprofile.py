"""cProfile of one config-5 (or config-1) solve after a warm-up solve: where the host time goes."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2409_09471_b200 as T
from paper_2409_09471_b200 import configs
which = sys.argv[1] if len(sys.argv) > 1 else "5"
C = configs.config5(0) if which == "5" else configs.config1()
dev = torch.device("cuda", 0)
cfg = T.SolverConfig(**C["cfg"], zero_rel=None, rounding="rto")
a = T.TTOperator(C["op"], device=dev); b = T.TTVector(C["b"], device=dev)
sk = T.kr_sketch_new(C["dims"], cfg.sketch_rows, seed=C["sketch_seed"], device=dev)
frame = T.make_solver_frame(b, cfg, seed=C["frame_seed"])
T.tt_sgmres(a, b, None, cfg, sk, frame); torch.cuda.synchronize()
t0 = time.perf_counter()
pr = cProfile.Profile(); pr.enable()
_, rep = T.tt_sgmres(a, b, None, cfg, sk, frame); torch.cuda.synchronize()
pr.disable()
print("wall", time.perf_counter() - t0, "iterations", rep.iterations)
st = pstats.Stats(pr); st.sort_stats("tottime").print_stats(25)
