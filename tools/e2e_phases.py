"""Where the host-buffer (e2e) step spends its time beyond the device-resident
step: events around the pipeline phases, host cores pinned (diagnostics)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2409_09471_b200 as T
from paper_2409_09471_b200 import configs, rto
dev = torch.device("cuda", 0)
C = configs.config3()
spec = T.RoundSpec(C["rel_tol"], C["max_rank"])
drm = [torch.as_tensor(g, device=dev) for g in C["drm"]]
host_op = [torch.as_tensor(g).pin_memory() for g in C["op"]]
host_x = [torch.as_tensor(c).pin_memory() for c in C["x"]]
opd = T.TTOperator(C["op"], device=dev); xd = T.TTVector(C["x"], device=dev)
oph = T.TTOperator(host_op); xh = T.TTVector(host_x)
st = torch.cuda.current_stream(dev)


def timed(f, reps=5):
    f(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps): f()
    b.record(st); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


print("device-resident step %.2f ms" % timed(lambda: T.tt_matvec_round_rto(opd, xd, spec, drm, device=dev)))
print("host step (e2e)      %.2f ms" % timed(lambda: T.tt_matvec_round_rto(oph, xh, spec, drm, device=dev)))
for ch in (1, 2, 4, 8):
    print("host step chunk %d   %.2f ms" % (ch, timed(lambda: T.tt_matvec_round_rto(oph, xh, spec, drm, chunk=ch, device=dev))))
# raw transfer times
bufs = [torch.empty(tuple(c.shape), dtype=torch.float64, device=dev) for c in host_op + host_x]
def h2d():
    for b, h in zip(bufs, host_op + host_x): b.copy_(h, non_blocking=True)
print("H2D 162 MB           %.2f ms" % timed(h2d))
outs = [torch.empty(64 * 128 * 64, dtype=torch.float64).pin_memory() for _ in range(30)]
src = torch.empty(64 * 128 * 64, dtype=torch.float64, device=dev)
def d2h():
    for o in outs: o.copy_(src, non_blocking=True)
print("D2H 126 MB           %.2f ms" % timed(d2h))
