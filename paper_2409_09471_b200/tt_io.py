"""TT containers, drop-in for the reference's save_vector / load_vector /
save_operator / load_operator (tt.py:451-520): magic "TTKVEC01" / "TTKOPR01",
int64 little-endian header, row-major float64 cores.  The file I/O is native
(csrc/tt_io.cu): cores stream between the file and device memory through two
pinned staging buffers.  A bad magic or a truncated file raises ValueError, as
in the reference (test_tt.py:382-387)."""

from __future__ import annotations

import ctypes
import os

import torch

from . import _lib
from .tt import TTOperator, TTVector, default_device


def _header_ints(header):
    return (ctypes.c_longlong * len(header))(*[int(x) for x in header])


def _write(path, kind, header, cores):
    lib = _lib.load()
    dev_mode = cores[0].is_cuda
    if dev_mode:
        st = _lib.stream_ptr(cores[0].device)
        cores = [c.contiguous() for c in cores]
    else:
        st = None
        cores = [c.contiguous().to(torch.float64) for c in cores]
    _lib.check(lib.ttk_io_write(os.fsencode(os.fspath(path)), kind, int(header[0]), _header_ints(header),
                                1 if dev_mode else 0, _lib.ptr_array(cores), st))


def read_header(path):
    """(kind, d, header ints) of a container; kind 0 = vector, 1 = operator."""
    lib = _lib.load()
    kind, d = ctypes.c_int(0), ctypes.c_int(0)
    buf = (ctypes.c_longlong * (3 * 4096 + 2))()
    _lib.check(lib.ttk_io_read_header(os.fsencode(os.fspath(path)), ctypes.byref(kind), ctypes.byref(d), buf,
                                      len(buf)))
    n = 1 + (2 if kind.value else 1) * d.value + d.value + 1
    return kind.value, d.value, [int(buf[i]) for i in range(n)]


def _read(path, want_kind, device):
    kind, d, h = read_header(path)
    if kind != want_kind:
        raise ValueError("not a TT " + ("operator" if want_kind else "vector") + " container")
    device = torch.device(device) if device is not None else default_device()
    if kind == 0:
        dims, ranks = h[1:1 + d], h[1 + d:2 + 2 * d]
        shapes = [(ranks[k], dims[k], ranks[k + 1]) for k in range(d)]
    else:
        rows, cols, ranks = h[1:1 + d], h[1 + d:1 + 2 * d], h[1 + 2 * d:2 + 3 * d]
        shapes = [(ranks[k], rows[k], cols[k], ranks[k + 1]) for k in range(d)]
    cores = [torch.empty(s, dtype=torch.float64, device=device) for s in shapes]
    lib = _lib.load()
    on_dev = device.type == "cuda"
    _lib.check(lib.ttk_io_read_cores(os.fsencode(os.fspath(path)), 1 if on_dev else 0, _lib.ptr_array(cores),
                                     _lib.stream_ptr(device) if on_dev else None))
    return cores


def save_vector(path, v: TTVector) -> None:
    """Write a TTVector to the binary container format (tt.py:466-474)."""
    _write(path, 0, [v.d] + list(v.dims) + list(v.ranks), list(v.cores))


def load_vector(path, device=None) -> TTVector:
    """Read a TTVector container onto `device` (default: cuda:0)."""
    return TTVector(_read(path, 0, device))


def save_operator(path, a: TTOperator) -> None:
    """Write a TTOperator to the binary container format (tt.py:493-502)."""
    _write(path, 1, [a.d] + list(a.row_dims) + list(a.col_dims) + list(a.ranks), list(a.op_cores))


def load_operator(path, device=None) -> TTOperator:
    """Read a TTOperator container onto `device` (default: cuda:0)."""
    return TTOperator(_read(path, 1, device))
