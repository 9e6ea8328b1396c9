"""Join a TTK_GEMM_TRACE log with an ncu launch list (same run): time and
TF/s per GEMM shape (diagnostics)."""
import csv, io, re, sys, collections
# one entry per launch: the problems of that launch (first one names the shape)
trace, cur = [], None
for l in open(sys.argv[1]):
    if l.startswith("gemm-launch"):
        cur = []
        trace.append(cur)
    elif l.startswith("gemm cfg=") and cur is not None:
        cur.append(l)
lines = [l for l in open(sys.argv[2]) if not l.startswith("==")]
rows = list(csv.DictReader(io.StringIO("".join(lines))))
g = [r for r in rows if r["Kernel Name"].startswith("void gemm_group_kernel") or r["Kernel Name"].startswith("gemm_splitk")]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
ti = 0
i = 0
while i < len(g) and ti < len(trace):
    r = g[i]
    if not r["Kernel Name"].startswith("void gemm_group_kernel"):
        i += 1
        continue
    t = trace[ti]
    m = dict(re.findall(r"(\w+)=(-?\d+)", t[0]))
    nprob = len(t)
    us = float(r["Metric Value"].replace(",", "")) / 1000
    red = 0.0
    if i + 1 < len(g) and g[i + 1]["Kernel Name"].startswith("gemm_splitk"):
        red = float(g[i + 1]["Metric Value"].replace(",", "")) / 1000
        i += 1
    key = (int(m["M"]), int(m["N"]), int(m["K"]), int(m["cfg"]), int(m["splits"]))
    a = agg[key]
    a[0] += 1; a[1] += us; a[2] += red
    a[3] += sum(2.0 * int(dict(re.findall(r"(\w+)=(-?\d+)", x))["M"]) * int(dict(re.findall(r"(\w+)=(-?\d+)", x))["N"])
                * int(dict(re.findall(r"(\w+)=(-?\d+)", x))["K"]) for x in t)
    ti += 1
    i += 1
tot = sum(a[1] + a[2] for a in agg.values())
print(f"total GEMM+reduce {tot/1e3:.2f} ms over {sum(a[0] for a in agg.values())} launches")
for k, a in sorted(agg.items(), key=lambda kv: -(kv[1][1] + kv[1][2])):
    n = a[0]
    print(f"M={k[0]:6d} N={k[1]:5d} K={k[2]:6d} cfg={k[3]} splits={k[4]:3d} n={n:4d} gemm {a[1]/n:7.1f} us + red {a[2]/n:6.1f} us = {(a[1]+a[2])/1e3:7.2f} ms  {a[3]/(a[1]+a[2])/1e6:6.2f} TF/s")
