import json,sys
d=json.loads(sys.stdin.read())
print(d["mode"], {k:(v["us"],v["sweeps"],"%.1e"%v["orth_v"],"%.1e"%v["sv_rel"]) for k,v in d.items() if k!="mode" and "error" not in v})
