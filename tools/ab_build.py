"""Build variant libraries for same-box A/B runs: ab/lib_<name>.so with extra
nvcc defines (diagnostics).  usage: python tools/ab_build.py name -DFOO=1 ..."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_09471_b200 import build as b
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
name, flags = sys.argv[1], sys.argv[2:]
out = os.path.join(root, "ab", f"lib_{name}.so")
os.makedirs(os.path.dirname(out), exist_ok=True)
print(b._compile(out, flags, os.path.join(root, "ab", f"build_{name}"), False))
