"""Build the native library libttk_b200.so in-tree with nvcc (sm_100a).

The .so is git-ignored but travels to the GPU box with the repo snapshot.
"""

from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG_DIR, "csrc")
INCLUDE = os.path.join(os.path.dirname(PKG_DIR), "include")
LIB_NAME = "libttk_b200.so"
LIB_PATH = os.path.join(PKG_DIR, LIB_NAME)

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "--expt-relaxed-constexpr",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: cannot build the sm_100a library")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale() -> bool:
    if not os.path.exists(LIB_PATH):
        return True
    t = os.path.getmtime(LIB_PATH)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(INCLUDE, "*.h"))
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, debug_knobs: bool = False, out: str | None = None) -> str:
    """Compile every csrc/*.cu into one shared library; returns its path.
    debug_knobs=True (experiments only) compiles the TTK_* environment knobs in
    and writes the library to `out` (never the shipped path)."""
    if debug_knobs:
        if not out or os.path.abspath(out) == LIB_PATH:
            raise ValueError("a debug-knob build needs its own output path")
        return _compile(out, ["-DTTK_DEBUG_KNOBS"], os.path.join(PKG_DIR, "build_dbg"), verbose)
    if not force and not _stale():
        return LIB_PATH
    return _compile(LIB_PATH, [], os.path.join(PKG_DIR, "build"), verbose)


def _compile(lib_path, extra, tmp_dir, verbose):
    objs = []
    nvcc = _nvcc()
    os.makedirs(tmp_dir, exist_ok=True)
    procs = []
    for src in sources():
        obj = os.path.join(tmp_dir, os.path.basename(src) + ".o")
        cmd = [nvcc, *[f for f in NVCC_FLAGS if f != "-shared"], *extra, "-c", "-I", INCLUDE, "-o", obj, src]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    failed = []
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            failed.append((src, out.decode(errors="replace")))
        elif verbose and out:
            print(out.decode(errors="replace"), file=sys.stderr)
    if failed:
        msg = "\n".join(f"--- {s}\n{o}" for s, o in failed)
        raise RuntimeError(f"nvcc failed:\n{msg}")
    tmp_lib = lib_path + ".tmp"
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
           "-o", tmp_lib, *objs]
    subprocess.run(cmd, check=True, capture_output=not verbose)
    os.replace(tmp_lib, lib_path)
    return lib_path


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
