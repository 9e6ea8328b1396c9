timeout 300 python bench.py --no-solver --no-cpu-baseline --steps 10 > gpurun_out/bench_q.json 2>gpurun_out/bench_q.err; echo bench=$?
python - <<'P'
import json
l=[x for x in open('gpurun_out/bench_q.json') if x.startswith('{')][-1]; d=json.loads(l)
print(round(d['value'],1), round(d['ms_per_step'],3), round(d['e2e']['value'],1), {k: round(v,3) for k,v in d['breakdown'].items()}, d['roofline']['dominant_kernel']['ms'])
P
