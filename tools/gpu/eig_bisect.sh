EIG_DBG=3 timeout 120 python tools/eig_one.py 80 50 2>&1 | grep "^info"
timeout 120 python tools/eig_one.py 80 64 50 128 33 2>&1 | grep "x"
