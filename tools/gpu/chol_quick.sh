python tools/subspace_one.py 2
python tools/chol_one.py 80
python tools/chol_one.py 50
python tools/qr_one.py 2>&1 | tail -3
