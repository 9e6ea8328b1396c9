"""TT containers (reference tt.py:451-520, test_tt.py:363-387) through the C ABI.

CPU tests use the host mode of the native reader/writer against files written
by the REFERENCE itself (tests/golden/make_golden.py gen_serial); GPU tests
round-trip device TTs, including cores larger than one pinned staging buffer."""

import ctypes
import os

import numpy as np
import pytest
import torch

from golden_io import load

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _lib():
    from paper_2409_09471_b200 import _lib as L
    return L, L.load()


def _host_read(path):
    L, lib = _lib()
    from paper_2409_09471_b200.tt_io import read_header
    kind, d, h = read_header(path)
    if kind == 0:
        dims, ranks = h[1:1 + d], h[1 + d:]
        shapes = [(ranks[k], dims[k], ranks[k + 1]) for k in range(d)]
    else:
        rows, cols, ranks = h[1:1 + d], h[1 + d:1 + 2 * d], h[1 + 2 * d:]
        shapes = [(ranks[k], rows[k], cols[k], ranks[k + 1]) for k in range(d)]
    cores = [np.empty(s, dtype=np.float64) for s in shapes]
    ptrs = (ctypes.c_void_p * d)(*[c.ctypes.data for c in cores])
    rc = lib.ttk_io_read_cores(os.fsencode(path), 0, ptrs, None)
    assert rc == 0, lib.ttk_last_error()
    return kind, h, cores


def _gold_cores(prefix):
    z = load("serial.npz")
    return [z[f"{prefix}__{k}"] for k in range(int(z[f"{prefix}__d"]))]


@pytest.mark.parametrize("name,kind,prefix", [("serial_vec.ttk", 0, "vec"), ("serial_op.ttk", 1, "op")])
def test_read_reference_files(name, kind, prefix):
    k, h, cores = _host_read(os.path.join(GOLD, name))
    assert k == kind
    for a, b in zip(cores, _gold_cores(prefix)):
        assert a.shape == b.shape and np.array_equal(a, b)


@pytest.mark.parametrize("name,kind,prefix", [("serial_vec.ttk", 0, "vec"), ("serial_op.ttk", 1, "op")])
def test_write_is_byte_identical_to_reference(tmp_path, name, kind, prefix):
    L, lib = _lib()
    cores = [np.ascontiguousarray(c) for c in _gold_cores(prefix)]
    d = len(cores)
    if kind == 0:
        header = [d] + [c.shape[1] for c in cores] + [1] + [c.shape[2] for c in cores]
    else:
        header = [d] + [c.shape[1] for c in cores] + [c.shape[2] for c in cores] + [1] + [c.shape[3] for c in cores]
    out = tmp_path / "w.ttk"
    ptrs = (ctypes.c_void_p * d)(*[c.ctypes.data for c in cores])
    hdr = (ctypes.c_longlong * len(header))(*header)
    rc = lib.ttk_io_write(os.fsencode(str(out)), kind, d, hdr, 0, ptrs, None)
    assert rc == 0, lib.ttk_last_error()
    assert out.read_bytes() == open(os.path.join(GOLD, name), "rb").read()


def test_magic_and_truncation_raise_valueerror(tmp_path):
    from paper_2409_09471_b200.tt_io import read_header
    junk = tmp_path / "junk.ttk"
    junk.write_bytes(b"NOTMAGIC" + b"\x00" * 64)
    with pytest.raises(ValueError):
        read_header(str(junk))
    good = open(os.path.join(GOLD, "serial_vec.ttk"), "rb").read()
    cut = tmp_path / "cut.ttk"
    cut.write_bytes(good[:-16])
    L, lib = _lib()
    kind, h, _ = _host_read(os.path.join(GOLD, "serial_vec.ttk"))
    cores = [np.empty((h[1 + 3 + k], h[1 + k], h[1 + 3 + k + 1])) for k in range(3)]
    ptrs = (ctypes.c_void_p * 3)(*[c.ctypes.data for c in cores])
    assert lib.ttk_io_read_cores(os.fsencode(str(cut)), 0, ptrs, None) == 2


@pytest.mark.gpu
def test_device_round_trip(tmp_path, cuda):
    import paper_2409_09471_b200 as T
    v = T.tt_random([7, 300, 5], [40, 500], seed=3, device=cuda)  # core 1: 40*300*500*8 B = 48 MB > staging
    T.save_vector(tmp_path / "v.ttk", v)
    w = T.load_vector(tmp_path / "v.ttk", device=cuda)
    assert w.dims == v.dims and w.ranks == v.ranks
    assert all(torch.equal(a, b) for a, b in zip(v.cores, w.cores))
    a = T.TTOperator([torch.randn(1, 3, 2, 4, dtype=torch.float64), torch.randn(4, 5, 6, 1, dtype=torch.float64)],
                     device=cuda)
    T.save_operator(tmp_path / "a.ttk", a)
    b = T.load_operator(tmp_path / "a.ttk", device=cuda)
    assert b.row_dims == a.row_dims and b.col_dims == a.col_dims
    assert all(torch.equal(x, y) for x, y in zip(a.op_cores, b.op_cores))
    # the device writer produces the reference's bytes
    gold = [torch.as_tensor(c, device=cuda) for c in _gold_cores("vec")]
    T.save_vector(tmp_path / "g.ttk", T.TTVector(gold))
    assert (tmp_path / "g.ttk").read_bytes() == open(os.path.join(GOLD, "serial_vec.ttk"), "rb").read()
