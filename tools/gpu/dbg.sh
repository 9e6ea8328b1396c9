for i in 1 2 3; do TTK_TMA_VERIFY=1 TTK_TMA_SMEM_PAD=150000 python tools/ab_run.py tools/inflight_repro.py 2 5 rto 2>&1 | grep -o "differing.*\|TMA GEMM mismatch.*" | head -8; echo; done
