timeout 600 python -m pytest tests/test_gpu_round.py -x -q -m gpu -k "rto" 2>&1 | tail -3
python tools/solver_profile.py 0 20 2>&1 | tail -1 | cut -c1-120
TTK_RTO_NO_DEFER=1 python tools/ab_run.py tools/solver_profile.py 0 20 2>&1 | tail -1 | cut -c1-120
python tools/solver_profile.py 0 20 2>&1 | tail -1 | cut -c1-120
bash tools/gpu/quick_bench.sh
