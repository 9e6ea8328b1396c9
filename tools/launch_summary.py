"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel."""
import csv, collections, io, sys

def load(path):
    lines = [l for l in open(path) if not l.startswith("==")]
    return list(csv.DictReader(io.StringIO("".join(lines))))

def summary(path, top=25):
    rows = load(path)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        name = r["Kernel Name"]
        name = name.split("(")[0][:70]
        v = float(r["Metric Value"].replace(",", ""))
        u = r["Metric Unit"]
        # to microseconds
        v = v / 1e3 if u in ("nsecond", "ns") else (v * 1e3 if u in ("msecond", "ms") else v)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    out = [f"launches={len(rows)} total_kernel_ms={tot/1e3:.3f}"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        out.append(f"{v[1]/1e3:9.3f} ms {100*v[1]/tot:5.1f}%  n={v[0]:5d}  avg={v[1]/v[0]:8.1f} us  {k}")
    return "\n".join(out)

if __name__ == "__main__":
    print(summary(sys.argv[1]))
