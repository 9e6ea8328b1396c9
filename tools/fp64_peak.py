"""Measure the FP64 roofline denominators on the GPU box (cuBLAS DGEMM via torch + host info)."""
import json, os, platform, subprocess, time
import torch

def dgemm(n=8192, reps=10):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    c = a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); c = a @ b; e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return 2 * n**3 / (best * 1e-3) / 1e12

def copy_bw(nbytes=4 << 30):
    a = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda").normal_()
    b = torch.empty_like(a)
    b.copy_(a); torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); b.copy_(a); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return 2 * nbytes / (best * 1e-3) / 1e9

out = {"dgemm_tflops_8192": dgemm(), "dgemm_tflops_4096": dgemm(4096), "copy_gbs_fp64": copy_bw(),
       "host_cores": os.cpu_count(), "cpu": platform.processor()}
try:
    out["cpu_model"] = [l for l in open("/proc/cpuinfo") if l.startswith("model name")][0].split(":")[1].strip()
except Exception:
    pass
print(json.dumps(out))
