set -x
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02b_pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/r02b_pytest_gpu.log
python bench.py > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err; echo bench=$?
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02b_bench_ref.json 2> gpurun_out/r02b_bench_ref.err; echo ref=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02b_launches_step.csv python tools/profile_step.py cfg3 2 > /dev/null 2>&1; echo launches=$?
python tools/launch_summary.py gpurun_out/r02b_launches_step.csv > gpurun_out/r02b_launches_step_summary.txt; cat gpurun_out/r02b_launches_step_summary.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:trunc_subspace -c 1 -o gpurun_out/r02b_trunc_subspace python tools/subspace_one.py 1 > /dev/null 2>&1; echo ncu_ss=$?
ncu -i gpurun_out/r02b_trunc_subspace.ncu-rep --page raw --csv > gpurun_out/r02b_trunc_subspace_raw.csv 2>/dev/null; echo raw=$?
python tools/qr_rto_phases.py 2>&1 | tail -3
