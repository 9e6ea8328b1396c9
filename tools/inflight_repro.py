"""Several host threads, each running config-3 work on its own stream (the
bench's in-flight mode), to reproduce concurrency faults (diagnostics):
python tools/inflight_repro.py nthreads steps mode   (mode: pipe | matvec | rto | trunc | seq)"""
import os, sys, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2409_09471_b200 as T
from paper_2409_09471_b200 import configs
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
mode = sys.argv[3] if len(sys.argv) > 3 else "pipe"
dev = torch.device("cuda", 0)
C = configs.config3()
op = T.TTOperator(C["op"], device=dev); x = T.TTVector(C["x"], device=dev)
drm = [torch.as_tensor(g, device=dev) for g in C["drm"]]
spec = T.RoundSpec(0.0, 64)
y0 = T.tt_matvec(op, x); lo0 = T.rto_sweeps(y0, drm); torch.cuda.synchronize()
def step():
    if mode == "pipe":
        return T.tt_matvec_round_rto(op, x, spec, drm, device=dev)
    if mode == "matvec":
        return T.tt_matvec(op, x)
    if mode == "rto":
        return T.rto_sweeps(y0, drm)
    if mode == "trunc":
        return T.tt_truncate_left_orth(lo0, spec)
    return T.tt_truncate_left_orth(T.rto_sweeps(T.tt_matvec(op, x), drm), spec)
ref = step(); torch.cuda.synchronize()
errs = []
LOCK = threading.Lock() if os.environ.get("REPRO_LOCK") else None
def locked_step():
    if LOCK is None:
        return step()
    with LOCK:
        return step()
def worker(i):
    try:
        torch.cuda.set_device(dev)
        s = torch.cuda.Stream(dev)
        with torch.cuda.stream(s):
            for _ in range(steps):
                y = locked_step()
            s.synchronize()
            diff = T.tt_add(y, T.tt_scale(ref, -1.0))
            print(i, "ok ranks", y.ranks == ref.ranks, "rel diff (tensor)", float(T.tt_norm(diff)) / float(T.tt_norm(ref)),
                  "max core diff", max(float((a - b).abs().max()) for a, b in zip(y.cores, ref.cores)),
                  "differing cores", [k for k, (a, b) in enumerate(zip(y.cores, ref.cores)) if float((a - b).abs().max()) > 1e-9][:8],
                  flush=True)
    except Exception as e:
        errs.append(e); print(i, "ERR", str(e)[-200:], flush=True)
from paper_2409_09471_b200 import _lib
if os.environ.get("REPRO_NO_TMA"):
    _lib.load().ttk_gemm_tma_enable(0)
ths = [threading.Thread(target=worker, args=(i,)) for i in range(n)]
[t.start() for t in ths]; [t.join() for t in ths]
print("errors", len(errs))
