EIG_DBG=3 timeout 120 python tools/eig_one.py 80 2>&1 | grep "^info\|x80"
timeout 300 ncu --set full --import-source on --clock-control none -k regex:gram_eig -c 1 -o gpurun_out/eig80c python tools/eig_one.py 80 > gpurun_out/ncu_eig.log 2>&1; tail -1 gpurun_out/ncu_eig.log
