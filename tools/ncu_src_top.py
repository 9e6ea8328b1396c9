"""Summarise an `ncu -i X --page source --csv --print-source sass` dump:
stall totals by reason and the top-N SASS lines by samples."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; data = rows[2:]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
ci = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = {r: 0 for r in reasons}
lines = []
for r in data:
    if len(r) < len(hdr):
        continue
    try:
        s = int(r[ci["# Samples"]] or 0)
    except ValueError:
        continue
    st = {}
    for k in reasons:
        try:
            v = int(r[ci[k]] or 0)
        except ValueError:
            v = 0
        tot[k] += v
        if v:
            st[k[6:]] = v
    lines.append((s, r[ci["Address"]], r[ci["Source"]], st))
print("total samples", sum(l[0] for l in lines))
print(sorted(((v, k) for k, v in tot.items() if v), reverse=True))
for s, a, src, st in sorted(lines, key=lambda t: -t[0])[:top]:
    print(f"{s:6d} {a:>6} {src[:60]:60s} {sorted(st.items(), key=lambda t: -t[1])[:3]}")
