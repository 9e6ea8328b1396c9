for k in 0 1 0 1; do
if [ $k = 1 ]; then export TTK_FQ_NOSYNC=1; else unset TTK_FQ_NOSYNC; fi
python tools/ab_run.py bench.py --no-solver --no-cpu-baseline --steps 10 2>/dev/null | python -c "
import json,sys
l=[x for x in sys.stdin if x.startswith('{')][-1]; d=json.loads(l)
print('nosync=$k', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['breakdown'].items()}, round(d['e2e']['ms_per_step'],3))"
done
