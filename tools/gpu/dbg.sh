for i in 1 2 3 4; do python tools/inflight_repro.py 2 5 pipe 2>&1 | grep -o "rel diff (tensor) [0-9.e-]*" | tr '\n' ' '; echo; done
for i in 1 2; do python tools/inflight_repro.py 3 4 rto 2>&1 | grep -o "rel diff (tensor) [0-9.e-]*" | tr '\n' ' '; echo; done
timeout 600 python -m pytest tests/test_gpu_baseline.py -x -q -m gpu -k "config3" 2>&1 | tail -3
