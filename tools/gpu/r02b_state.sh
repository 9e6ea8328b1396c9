set -x
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_step.csv python tools/profile_step.py cfg3 2 > gpurun_out/ncu_launch.log 2>&1; echo rc=$?; tail -2 gpurun_out/ncu_launch.log
python tools/launch_summary.py gpurun_out/launches_step.csv
