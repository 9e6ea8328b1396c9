"""Run a tool against the debug-knob library build (ab/libttk_dbg.so, TTK_* knobs honoured):
    python tools/ab_run.py tools/jac_time.py 80"""
import os, runpy, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_09471_b200 import _lib
_lib.LIB_PATH = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "ab", "libttk_dbg.so")
sys.argv = sys.argv[1:]
runpy.run_path(sys.argv[0], run_name="__main__")
