timeout 900 python -m pytest tests/test_gpu_round.py tests/test_gpu_baseline.py -x -q -m gpu 2>&1 | tail -5
timeout 300 python bench.py --no-solver --no-cpu-baseline --steps 10 > gpurun_out/bench_gram.json 2>gpurun_out/bench_gram.err; echo bench=$?
python - <<'P'
import json
l=[x for x in open('gpurun_out/bench_gram.json') if x.startswith('{')][-1]; d=json.loads(l)
print(d['value'], d['ms_per_step'], d['e2e']['value'], d.get('parity'), d.get('breakdown'))
P
