"""DMMA grouped GEMM through the C ABI (ttk_gemm_strided) over the tile menu:
every shape family the rounding/sketch paths launch (tall-skinny rank-80
products, Gram matrices with split-K, 80-row carries times wide cores) against
a float64 torch reference.  Tolerance: |C - C_ref| <= 1e-13 * (|A| |B|)_max * sqrt(K)."""

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

# (M, N, K, layout) -- layout "nn": A row-major (m,k), B row-major (k,n);
# "tn": A stored k-major (A^T row-major), "nt": B stored n-major
SHAPES = [
    (24576, 80, 192, "nn"),   # RTO right partial contraction (64x80 tiles, no split)
    (10240, 80, 192, "nn"),   # sketch of a projected core (64x80, split 2)
    (80, 80, 10240, "tn"),    # Gram matrix (80x80 tile, split-K)
    (80, 192, 10240, "tn"),   # carry projection (80x64 tiles, split-K)
    (192, 80, 10240, "nt"),   # 64x80 / split
    (80, 24576, 192, "nn"),   # carry times core (80x64 tiles)
    (64, 8192, 80, "tn"),
    (8192, 80, 80, "tn"),
    (80, 80, 80, "nn"),
    (4096, 384, 128, "nn"),   # matvec-like (128x128)
    (1000, 70, 33, "nn"),     # ragged edges
    (7, 5, 3, "nn"),
]


def _strides(M, N, K, layout):
    if layout == "nn":
        return (K, 1), (N, 1)            # a_ms, a_ks ; b_ks, b_ns
    if layout == "tn":
        return (1, M), (N, 1)
    return (K, 1), (1, K)                # nt


@pytest.mark.parametrize("M,N,K,layout", SHAPES)
@pytest.mark.parametrize("beta", [0.0, 0.5])
def test_gemm_strided_shapes(native_lib, cuda, M, N, K, layout, beta):
    from paper_2409_09471_b200 import _lib
    g = torch.Generator().manual_seed(M * 7 + N * 3 + K)
    A = torch.randn(M * K, dtype=torch.float64, generator=g)
    B = torch.randn(K * N, dtype=torch.float64, generator=g)
    C0 = torch.randn(M * N, dtype=torch.float64, generator=g)
    (a_ms, a_ks), (b_ks, b_ns) = _strides(M, N, K, layout)
    Am = torch.as_strided(A, (M, K), (a_ms, a_ks))
    Bm = torch.as_strided(B, (K, N), (b_ks, b_ns))
    ref = 1.5 * (Am @ Bm) + beta * C0.view(M, N)
    dA, dB, dC = A.to(cuda), B.to(cuda), C0.to(cuda).clone()
    ws_bytes = native_lib.ttk_gemm_strided_ws_bytes(1, M, N, K)
    ws = _lib.workspace(max(int(ws_bytes), 8), cuda)
    rc = native_lib.ttk_gemm_strided(1, M, N, K, 1.5, dA.data_ptr(), a_ms, a_ks, 0, dB.data_ptr(), b_ks, b_ns, 0,
                                     beta, dC.data_ptr(), N, 1, 0, ws.data_ptr(), ws.numel(),
                                     _lib.stream_ptr(cuda))
    assert rc == 0, native_lib.ttk_last_error()
    torch.cuda.synchronize()
    err = (dC.cpu().view(M, N) - ref).abs().max().item()
    scale = 1.5 * Am.abs().max().item() * Bm.abs().max().item() * math.sqrt(K)
    assert err <= 1e-13 * scale * math.sqrt(K) + 1e-300, (err, scale)


def test_gemm_split_reduce_deterministic(native_lib, cuda):
    """Split-K partial sums are reduced in a fixed order: two runs are bitwise equal."""
    from paper_2409_09471_b200 import _lib
    M, N, K = 80, 80, 10240
    g = torch.Generator().manual_seed(5)
    A = torch.randn(K, M, dtype=torch.float64, generator=g).to(cuda)
    outs = []
    for _ in range(2):
        C = torch.empty(M, N, dtype=torch.float64, device=cuda)
        ws = _lib.workspace(int(native_lib.ttk_gemm_strided_ws_bytes(1, M, N, K)), cuda)
        rc = native_lib.ttk_gemm_strided(1, M, N, K, 1.0, A.data_ptr(), 1, M, 0, A.data_ptr(), M, 1, 0, 0.0,
                                         C.data_ptr(), N, 1, 0, ws.data_ptr(), ws.numel(), _lib.stream_ptr(cuda))
        assert rc == 0
        outs.append(C.cpu().numpy())
    assert np.array_equal(outs[0], outs[1])
    ref = (A.cpu().T @ A.cpu()).numpy()
    assert np.abs(outs[0] - ref).max() <= 1e-12 * np.abs(ref).max()


@pytest.mark.parametrize("cfg", list(range(12)))
def test_gemm_every_tile_config(cfg):
    """Each tile configuration of the grouped GEMM (forced through
    TTK_GEMM_FORCE_CFG in a subprocess) on ragged shapes in three layouts."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, TTK_GEMM_FORCE_CFG=str(cfg))
    out = subprocess.run([sys.executable, os.path.join(root, "tools", "gemm_check.py")], env=env,
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("cfg=")]
    assert len(lines) == 15, out.stdout
    bad = [l for l in lines if "BAD" in l or "rc=0" not in l]
    assert not bad, "\n".join(bad)
