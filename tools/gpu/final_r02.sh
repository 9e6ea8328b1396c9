set -x
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02c_pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/r02c_pytest_gpu.log
python bench.py > gpurun_out/r02c_bench.json 2> gpurun_out/r02c_bench.err; echo bench=$?
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02c_bench_ref.json 2> gpurun_out/r02c_bench_ref.err; echo ref=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02c_launches_step.csv python tools/profile_step.py cfg3 2 > /dev/null 2>&1; echo launches=$?
python tools/launch_summary.py gpurun_out/r02c_launches_step.csv > gpurun_out/r02c_launches_step_summary.txt; cat gpurun_out/r02c_launches_step_summary.txt
python __graft_entry__.py 2>&1 | tail -1
python tools/overlap_tma_grouped.py 3 | tail -1
