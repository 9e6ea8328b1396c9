"""B200-native (sm_100a, fp64) hot path of randomized TT-sGMRES (arXiv 2409.09471).

Drop-in mirror of the reference package ``ttkrylov``'s TT core-list API for the
path named by BASELINE.json: TT matvec, TT-axpy/concatenation, dot/norm,
TT-SVD and randomize-then-orthogonalize rounding, the Khatri-Rao sketch, the
streaming sketches and ``tt_sgmres``.  Cores are CUDA fp64 torch tensors; the
arithmetic runs in libttk_b200.so (C ABI: include/ttk_b200.h).
"""

from .errors import DegenerateRecovery, ShapeMismatch, SizeLimit
from .precond import (
    ExpSumPreconditioner,
    matrix_exp,
    mode_multiply,
    precond_apply,
)
from .rto import (CounterDRM, rto_flops, rto_ranks, rto_sweeps, tt_matvec_round_rto, tt_round_rto,
                  tt_truncate_left_orth)
from .sketch import (KhatriRaoSketch, kr_apply, kr_apply_batch, kr_apply_device, kr_apply_matvec,
                     kr_apply_matvec_device, kr_apply_rows, kr_sketch_new)
from .solvers import (
    PHASES,
    SolveReport,
    SolverConfig,
    make_solver_frame,
    sketched_lsq,
    solver_rto_drm,
    true_residual,
    tt_sgmres,
    tt_spgmres,
)
from .streaming import (
    PINV_RCOND,
    TTDRM,
    SketchPair,
    StreamFrame,
    combine_pairs,
    stream_recover,
    stream_sketch,
    tt_drm_new,
)
from .tt import (
    DENSE_CAP,
    ZERO_REL,
    RoundSpec,
    TTOperator,
    TTVector,
    attainable_ranks,
    identity_operator,
    kron_sum_operator,
    max_rank,
    tt_add,
    tt_combine,
    tt_dot,
    tt_dots,
    tt_matvec,
    tt_norm,
    tt_norm_left_orthogonal,
    tt_norm_orthogonal,
    tt_op_to_dense,
    tt_random,
    tt_rank_one,
    tt_round,
    tt_scale,
    tt_to_dense,
    tt_zero,
)

from .tt_io import load_operator, load_vector, read_header, save_operator, save_vector

__version__ = "0.1.0"
