python tools/solver_profile.py 0 20 2>&1 | tail -2
TTK_HOST_PROF=1 python tools/ab_run.py tools/solver_profile.py 0 20 2>&1 | tail -2
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5.csv python tools/solver_profile.py 0 6 > /dev/null 2>&1; python tools/launch_summary.py gpurun_out/launches_cfg5.csv | head -30
