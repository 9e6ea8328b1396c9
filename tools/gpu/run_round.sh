timeout 900 python -m pytest tests/test_gpu_round.py tests/test_gpu_baseline.py -x -q -m gpu 2>&1 | tail -4
bash tools/gpu/quick_bench.sh
