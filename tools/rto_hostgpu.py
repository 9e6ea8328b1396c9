"""Config-3 RTO sweeps: host issue time of the ttk_rto_sweeps call vs its GPU time,
and the number of kernels it launches (is the sweep host- or GPU-bound?)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2409_09471_b200 as T
from paper_2409_09471_b200 import configs, _lib
dev = torch.device("cuda", 0)
C3 = configs.config3()
op, x = T.TTOperator(C3["op"], device=dev), T.TTVector(C3["x"], device=dev)
y = T.tt_matvec(op, x)
drm = [torch.as_tensor(g, device=dev) for g in C3["drm"]]
lib = _lib.load()
for _ in range(3):
    T.rto_sweeps(y, drm)
torch.cuda.synchronize()
res = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n0 = lib.ttk_launch_count()
    e0.record(); t0 = time.perf_counter()
    T.rto_sweeps(y, drm)
    t1 = time.perf_counter(); e1.record(); torch.cuda.synchronize(); t2 = time.perf_counter()
    res.append({"host_issue_ms": (t1 - t0) * 1e3, "gpu_ms": e0.elapsed_time(e1), "wall_ms": (t2 - t0) * 1e3,
                "launches": lib.ttk_launch_count() - n0})
print(json.dumps(res))
