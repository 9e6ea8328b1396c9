"""CPU oracle for the TT-sGMRES hot path -- TEST INFRASTRUCTURE ONLY.

This package restates, in plain numpy, the reference algorithms of
``ttkrylov`` (arXiv 2409.09471 companion code, /root/reference/pkg/src) that
the B200 kernels replace.  Every function cites the reference file:line it
follows.  It is the parity checker used by ``tests/``, by
``__graft_entry__.smoke()`` and by the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py``; the product path (``paper_2409_09471_b200``) never
imports it.

Pinning: ``tests/test_oracle_golden.py`` checks every restated function
against golden vectors produced by running the reference itself in the build
container (``tests/golden/make_golden.py``).  The randomize-then-orthogonalize
rounding (``rto_round``) has no reference implementation; it is
pinned by the exactness known-answer test and dense oracles instead.
"""

from .ttoracle import *  # noqa: F401,F403
