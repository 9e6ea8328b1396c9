"""CPU checks of the drop-in boundary: the C-ABI library builds, loads and
exports every symbol declared in include/ttk_b200.h (no compute calls)."""

import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ttk_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ttk_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for required in ("ttk_matvec", "ttk_kr_sketch", "ttk_tt_concat", "ttk_tt_dots", "ttk_last_error"):
        assert required in syms


def test_library_exports_every_declared_symbol(native_lib):
    missing = [s for s in declared_symbols() if not hasattr(native_lib, s)]
    assert not missing, f"symbols declared in ttk_b200.h but not exported: {missing}"


def test_python_binding_covers_header(native_lib):
    from paper_2409_09471_b200 import _lib
    missing = [s for s in declared_symbols() if s not in _lib.SIGNATURES]
    assert not missing, f"no ctypes signature for {missing}"


def test_version_and_error_channel(native_lib):
    assert native_lib.ttk_version() == 1
    assert isinstance(native_lib.ttk_last_error(), bytes)


def test_library_is_sm100a():
    """The fatbin carries sm_100a SASS (cuobjdump)."""
    import subprocess
    from paper_2409_09471_b200 import build
    path = build.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", path], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
