#!/bin/bash
# compute-sanitizer runs over the kernels with intra-CTA / cluster hand-offs
# (race detection).  Logs under profiles/ (r02_sanitizer_*.log).
set -u
out=${1:-gpurun_out}
mkdir -p "$out"
CS=/usr/local/cuda/bin/compute-sanitizer
run() {  # name tool args...
  local name=$1 tool=$2; shift 2
  timeout 900 $CS --tool "$tool" --print-limit 20 "$@" > "$out/r02_sanitizer_${name}.log" 2>&1
  echo "exit=$?" >> "$out/r02_sanitizer_${name}.log"
  tail -3 "$out/r02_sanitizer_${name}.log"
}
# one-warp cluster Jacobi (80 x 80, DSMEM st.async + mbarrier block moves)
run racecheck_jacobi_warp racecheck python tools/jac_one.py 80
# 16-lane block Jacobi (rows > 96 -> jacobi_block_kernel), 112 x 112
run racecheck_jacobi_block racecheck python tools/jac_one.py 112
# fused CholeskyQR2 (cooperative grid barriers): synccheck + racecheck
run synccheck_cholqr2_fused synccheck python tools/qr_one.py
run racecheck_cholqr2_fused racecheck python tools/qr_one.py
# memcheck over the whole smoke path (matvec, RTO rounding, KR sketch)
run memcheck_smoke memcheck python __graft_entry__.py
