"""ctypes binding of the C ABI declared in include/ttk_b200.h.

The product path has no CPU fallback: if libttk_b200.so is missing or no CUDA
device is present, every compute entry point raises.
"""

from __future__ import annotations

import ctypes
import os

import torch

from .errors import DegenerateRecovery, ShapeMismatch

_PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG_DIR, "libttk_b200.so")

c_int = ctypes.c_int
c_ll = ctypes.c_longlong
c_double = ctypes.c_double
c_size = ctypes.c_size_t
c_vp = ctypes.c_void_p
P_int = ctypes.POINTER(ctypes.c_int)
P_vp = ctypes.POINTER(ctypes.c_void_p)
P_double = ctypes.POINTER(ctypes.c_double)

# name -> (restype, argtypes); every symbol here is declared in include/ttk_b200.h
SIGNATURES = {
    "ttk_last_error": (ctypes.c_char_p, []),
    "ttk_version": (c_int, []),
    "ttk_device_arch": (c_int, []),
    "ttk_launch_count": (c_ll, []),
    "ttk_gemm_strided": (c_int, [c_int, c_int, c_int, c_int, c_double, c_vp, c_ll, c_ll, c_ll,
                                 c_vp, c_ll, c_ll, c_ll, c_double, c_vp, c_ll, c_ll, c_ll,
                                 c_vp, c_size, c_vp]),
    "ttk_gemm_strided_ws_bytes": (c_size, [c_int, c_int, c_int, c_int]),
    "ttk_matvec": (c_int, [c_int, P_int, P_int, P_int, P_int, P_vp, P_vp, P_vp, c_vp]),
    "ttk_matvec_range": (c_int, [c_int, P_int, P_int, P_int, P_int, P_vp, P_vp, P_vp, c_int, c_int, c_vp]),
    "ttk_matvec_banded": (c_int, [c_int, P_int, P_int, P_int, c_int, P_vp, ctypes.c_char_p, P_vp, P_vp, c_vp]),
    "ttk_mode_multiply": (c_int, [c_int, c_int, P_int, P_int, P_int, P_double, P_vp, P_vp, P_vp, c_vp]),
    "ttk_tt_concat": (c_int, [c_int, c_int, P_double, P_int, P_int, P_vp, P_vp, c_vp]),
    "ttk_scale": (c_int, [c_vp, c_vp, c_ll, c_double, c_vp]),
    "ttk_sumsq": (c_int, [c_vp, c_ll, c_vp, c_vp, c_size, c_vp]),
    "ttk_tt_dots": (c_int, [c_int, P_int, P_int, P_vp, c_int, P_int, P_vp, c_vp, c_vp, c_size, c_vp]),
    "ttk_tt_dots_ws_bytes": (c_size, [c_int, P_int, P_int, c_int, P_int]),
    "ttk_kr_sketch": (c_int, [c_int, P_int, c_int, c_int, P_vp, c_int, P_int, P_vp, c_vp, c_vp,
                              c_size, c_vp]),
    "ttk_kr_sketch_path": (c_int, [c_int, c_int, P_int, c_int, c_int, P_vp, c_int, P_int, P_vp, c_vp,
                                   c_vp, c_size, c_vp]),
    "ttk_kr_sketch_matvec": (c_int, [c_int, P_int, c_int, P_vp, P_int, P_int, P_vp, c_vp, c_vp, c_size, c_vp]),
    "ttk_kr_sketch_matvec_ws_bytes": (c_size, [c_int, c_int, P_int, P_int]),
    "ttk_debug_fused_qr_profile": (c_int, [c_vp]),
    "ttk_kr_sketch_ws_bytes": (c_size, [c_int, P_int, c_int, c_int, c_int, P_int]),
}

_lib = None


def load():
    """Load (once) and return the native library; raises if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"native library {LIB_PATH} is not built; run `python -m paper_2409_09471_b200.build` "
            "or __graft_entry__.build() (there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name, None)
        if fn is None:
            continue  # reported by tests/test_abi.py
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status: int):
    if status == 0:
        return
    msg = load().ttk_last_error().decode(errors="replace")
    if status == 1:
        raise ShapeMismatch(msg)
    if status == 2:
        raise ValueError(msg)
    if status == 5:
        raise DegenerateRecovery(msg)
    raise RuntimeError(f"ttk native error {status}: {msg}")


def require_cuda(t: torch.Tensor, what: str = "tensor"):
    if not t.is_cuda:
        raise RuntimeError(f"{what} must live on a CUDA device: the B200 path has no CPU fallback")


def int_array(vals):
    vals = [int(v) for v in vals]
    return (ctypes.c_int * max(len(vals), 1))(*vals)


def double_array(vals):
    vals = [float(v) for v in vals]
    return (ctypes.c_double * max(len(vals), 1))(*vals)


def ptr_array(tensors):
    ptrs = [t.data_ptr() if t is not None else 0 for t in tensors]
    return (ctypes.c_void_p * max(len(ptrs), 1))(*ptrs)


def stream_ptr(device=None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


_WORKSPACES = {}


def workspace(nbytes: int, device) -> torch.Tensor:
    """Scratch for one ABI call: a view of a grow-only buffer kept per
    (device, current stream).  Every wrapper uses one workspace per call and the
    calls on a stream are ordered, so reuse is safe; allocating a fresh tensor
    per call made the caching allocator fall through to cudaMalloc (which
    synchronises the device) whenever the sizes changed -- every solver
    iteration."""
    dev = torch.device(device)
    n = max(int(nbytes), 256)
    if dev.type != "cuda":
        return torch.empty(n, dtype=torch.uint8, device=dev)
    key = (dev.index if dev.index is not None else torch.cuda.current_device(),
           torch.cuda.current_stream(dev).cuda_stream)
    buf = _WORKSPACES.get(key)
    if buf is None or buf.numel() < n:
        grow = n if buf is None else max(n, buf.numel() + buf.numel() // 2)
        _WORKSPACES.pop(key, None)
        buf = torch.empty(grow, dtype=torch.uint8, device=dev)
        _WORKSPACES[key] = buf
    return buf[:n]

SIGNATURES.update({
    "ttk_qr": (c_int, [c_int, c_int, c_vp, c_ll, c_ll, c_vp, c_ll, c_ll, c_vp, c_vp, c_size, c_vp]),
    "ttk_qr_ws_bytes": (c_size, [c_int, c_int]),
    "ttk_svd_small": (c_int, [c_int, c_int, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "ttk_gemm_tma": (c_int, [c_int, c_int, c_int, c_double, c_vp, c_ll, c_vp, c_ll, c_double, c_vp, c_ll, c_vp]),
    "ttk_gemm_tma_strided": (c_int, [c_int, c_int, c_int, c_double, c_vp, c_ll, c_ll, c_vp, c_ll, c_ll, c_double,
                                     c_vp, c_ll, c_ll, c_vp, c_size, c_vp]),
    "ttk_tt_round": (c_int, [c_int, P_int, P_int, P_vp, c_double, c_int, c_double, P_vp, P_int, c_vp,
                             c_size, c_vp]),
    "ttk_tt_round_ws_bytes": (c_size, [c_int, P_int, P_int]),
    "ttk_rto_sweeps": (c_int, [c_int, P_int, P_int, P_vp, P_int, P_vp, P_vp, c_vp, c_size, c_vp]),
    "ttk_rto_sweeps_ev": (c_int, [c_int, P_int, P_int, P_vp, P_int, P_vp, P_vp, c_vp, c_size, P_vp, c_vp]),
    "ttk_rto_ws_bytes": (c_size, [c_int, P_int, P_int, P_int]),
})

SIGNATURES.update({
    "ttk_stream_sketch": (c_int, [c_int, P_int, P_int, P_vp, P_int, P_vp, P_int, P_vp, P_vp, P_vp, c_vp,
                                  c_size, c_vp]),
    "ttk_stream_sketch_ws_bytes": (c_size, [c_int, P_int, P_int, P_int, P_int]),
    "ttk_axpy_multi": (c_int, [c_int, P_double, P_vp, c_ll, c_vp, c_vp]),
    "ttk_stream_recover_cores": (c_int, [c_int, P_int, P_int, P_int, P_vp, P_vp, c_double, P_vp, P_int,
                                         ctypes.POINTER(ctypes.c_int), c_vp, c_size, c_vp]),
    "ttk_stream_recover_ws_bytes": (c_size, [c_int, P_int, P_int, P_int]),
})

SIGNATURES.update({
    "ttk_debug_truncate_paths": (c_int, [c_vp]),
    "ttk_debug_truncate_paths_ex": (c_int, [c_vp, c_int]),
    "ttk_tt_truncate": (c_int, [c_int, P_int, P_int, P_vp, c_double, c_int, P_vp, P_int, c_vp, c_size, c_vp]),
    "ttk_tt_truncate_host": (c_int, [c_int, P_int, P_int, P_vp, c_double, c_int, P_vp, P_int, P_vp, c_vp, c_size,
                                     c_vp]),
    "ttk_tt_truncate_ws_bytes": (c_size, [c_int, P_int, P_int]),
})

SIGNATURES.update({"ttk_debug_svd_sweeps": (c_int, [c_vp])})
SIGNATURES.update({"ttk_debug_jacobi_profile": (c_int, [c_vp])})
SIGNATURES.update({
    "ttk_io_read_header": (c_int, [ctypes.c_char_p, P_int, P_int, ctypes.POINTER(ctypes.c_longlong), c_int]),
    "ttk_io_read_cores": (c_int, [ctypes.c_char_p, c_int, P_vp, c_vp]),
    "ttk_io_write": (c_int, [ctypes.c_char_p, c_int, c_int, ctypes.POINTER(ctypes.c_longlong), c_int, P_vp, c_vp]),
})
SIGNATURES.update({"ttk_debug_host_profile": (c_int, [ctypes.POINTER(ctypes.c_longlong)])})
SIGNATURES.update({"ttk_drm_gaussian": (c_int, [ctypes.c_ulonglong, c_int, c_int, c_int, c_int, c_int, c_int,
                                                c_double, c_vp, c_vp])})
SIGNATURES.update({"ttk_debug_chol_profile": (c_int, [c_vp])})
SIGNATURES.update({"ttk_debug_chol": (c_int, [c_int, c_vp, c_vp, c_vp, c_vp])})

SIGNATURES.update({"ttk_qr_auto": (c_int, [c_int, c_int, c_vp, c_ll, c_ll, c_vp, c_ll, c_ll, c_vp, c_vp, c_size,
                                           c_vp])})
SIGNATURES.update({"ttk_debug_trunc_subspace": (c_int, [c_int, c_int, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp])})
SIGNATURES.update({"ttk_gemm_tma_enable": (c_int, [c_int])})
SIGNATURES.update({"ttk_debug_occupy": (c_int, [c_int, c_int, c_int, c_ll, c_int, c_vp, c_vp, c_vp])})


class concurrent_problems:
    """Context for callers that keep several independent problems in flight on
    different CUDA streams: the sweeps use the cp.async grouped GEMM instead of
    the TMA-staged one while it is active (ttk_gemm_tma_enable, DESIGN 6.2)."""

    def __enter__(self):
        self._prev = load().ttk_gemm_tma_enable(0)
        return self

    def __exit__(self, *exc):
        load().ttk_gemm_tma_enable(self._prev)
        return False
