echo "== in-flight, production (guard + fixed kernel), x15"
for i in 1 2 3 4 5 6 7 8 9 10 11 12 13 14 15; do python tools/inflight_repro.py 2 4 pipe 2>&1 | grep -o "rel diff (tensor) [0-9.e-]*" | tr '\n' ' '; echo; done
echo "== explicit switch x10"
for i in 1 2 3 4 5 6 7 8 9 10; do REPRO_NO_TMA=1 python tools/inflight_repro.py 2 4 pipe 2>&1 | grep -o "rel diff (tensor) [0-9.e-]*" | tr '\n' ' '; echo; done
