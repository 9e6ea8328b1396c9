set -x
python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo bench=$?
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02_bench_ref.json 2> gpurun_out/r02_bench_ref.err; echo ref=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_step.csv python tools/profile_step.py cfg3 2 > /dev/null 2>&1; echo launches=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:jacobi_warp -c 1 -o gpurun_out/r02_jacobi_nov python tools/jac_one.py 80 nov > /dev/null 2>&1; echo jac=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_group -c 2 -o gpurun_out/r02_gemm_rto python tools/gemm_rto_shapes.py 24576x80x192 80x24576x192 > /dev/null 2>&1; echo gemm=$?
