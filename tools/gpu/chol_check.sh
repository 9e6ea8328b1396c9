set -x
python tools/subspace_one.py 2
python tools/chol_one.py 80
python tools/chol_one.py 64
python tools/chol_one.py 50
python tools/qr_one.py 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_round.py tests/test_gpu_baseline.py -x -q -m gpu 2>&1 | tail -5
bash tools/gpu/quick_bench.sh
