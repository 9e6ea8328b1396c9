set -x
timeout 900 python -m pytest tests/test_gpu_round.py -x -q -m gpu -k "truncate or round or rto" > gpurun_out/ss_round.log 2>&1; echo round=$?; tail -15 gpurun_out/ss_round.log
timeout 900 python -m pytest tests/test_gpu_baseline.py -x -q -m gpu -k "config3 or config2" > gpurun_out/ss_base.log 2>&1; echo base=$?; tail -15 gpurun_out/ss_base.log
bash tools/gpu/quick_bench.sh
