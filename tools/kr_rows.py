"""Config-4 Khatri-Rao sketch per-row throughput: the full s = 512 rows vs one
G-way row shard (64 rows at G = 8, 128 at G = 4, ...), one GPU."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2409_09471_b200 as T
from paper_2409_09471_b200 import configs
dev = torch.device("cuda", 0)
C = configs.config4()
sk = T.KhatriRaoSketch(C["factors"], device=dev)
vs = [T.TTVector(v, device=dev) for v in C["vecs"]]
del C
st = torch.cuda.current_stream(dev)
full = T.kr_apply_batch(sk, vs)
res = {}
for rows in (512, 256, 128, 64):
    for _ in range(2):
        part = T.kr_apply_rows(sk, vs, 0, rows)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(3):
        T.kr_apply_rows(sk, vs, 0, rows)
    b.record(st)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 3
    flops = 64 * sum(2.0 * rows * 64 * r0 * r1 for r0, r1 in zip([1] + [100] * 19, [100] * 19 + [1]))
    err = float((torch.linalg.norm(part - full[:, :rows], dim=1) / torch.linalg.norm(full[:, :rows], dim=1)).max())
    res[rows] = {"ms": round(ms, 3), "tflops": round(flops / ms / 1e9, 2), "rows_per_ms": round(rows / ms, 2),
                 "max_rel_diff_vs_full": err}
base = res[512]["rows_per_ms"]
for r in res:
    res[r]["per_row_vs_full"] = round(res[r]["rows_per_ms"] / base, 3)
print(json.dumps(res))
