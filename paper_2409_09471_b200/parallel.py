"""Multi-GPU partitioning of the hot path (one process per GPU, torch.distributed).

Only the two workloads that shard naturally are distributed:

* Khatri-Rao sketch rows (config 4): rank g owns rows [lo_g, hi_g) of every
  factor, sketches all vectors for its rows (no data-path collective), and
  one all-gather of the (B x s/G) row blocks reassembles the sketch in the
  reference's fixed row order (SPEC: "kr_apply rows may be computed
  independently ... fixed row positions").  Over NCCL this is a few-KB
  gather across NVLink/NVSwitch.
* Independent right-hand sides (config 5): RHS j is solved on rank j mod G;
  SolveReports are gathered on the host (no device collective).

matvec / rounding / a single solve do not shard: those run as replicas.
The partition and gather logic is backend-agnostic (tests run it with gloo
on CPU; bench.py runs it with NCCL).
"""

from __future__ import annotations

import time

import torch
import torch.distributed as dist


def row_partition(rows: int, world: int):
    """Balanced contiguous row blocks [(lo, hi)] covering [0, rows) in rank order."""
    base, extra = divmod(rows, world)
    out, lo = [], 0
    for g in range(world):
        hi = lo + base + (1 if g < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


def gather_row_blocks(block: torch.Tensor, parts, group=None) -> torch.Tensor:
    """All-gather per-rank (B x (hi-lo)) blocks into the full (B x rows) matrix,
    rows in fixed global order.  Blocks are padded to the largest width so a
    single all_gather works for uneven splits."""
    world = len(parts)
    width = max(hi - lo for lo, hi in parts)
    nb = block.shape[0]
    padded = torch.zeros((nb, width), dtype=block.dtype, device=block.device)
    padded[:, : block.shape[1]] = block
    bufs = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(bufs, padded.contiguous(), group=group)
    return torch.cat([b[:, : hi - lo] for b, (lo, hi) in zip(bufs, parts)], dim=1)


def kr_apply_sharded(sketch, vectors, rank: int, world: int, group=None, compute=None) -> torch.Tensor:
    """Sketch of every vector with the rows split over `world` ranks.

    compute(lo, hi) -> (B x (hi-lo)) tensor defaults to the device kernel
    (kr_apply_rows); tests inject the CPU oracle to exercise the gather on gloo."""
    parts = row_partition(sketch.rows, world)
    lo, hi = parts[rank]
    if compute is None:
        from .sketch import kr_apply_rows
        block = kr_apply_rows(sketch, vectors, lo, hi)
    else:
        block = compute(lo, hi)
    if world == 1:
        return block
    return gather_row_blocks(block, parts, group=group)


def rhs_assignment(n_rhs: int, world: int, rank: int):
    """RHS indices solved by `rank` (j mod world == rank)."""
    return [j for j in range(n_rhs) if j % world == rank]


def _run_concurrently(jobs, solve_one, concurrency: int, device):
    """Run solve_one(j) for every j in `jobs`, `concurrency` at a time, each on
    its own CUDA stream driven by its own host thread.  The solves are
    independent; one solve keeps the GPU busy only a fraction of the time (its
    per-core rank / path decisions synchronise the host), so concurrent
    streams fill the gaps.  ctypes releases the GIL inside the native calls and
    the library keys its scratch by stream.  Results are identical to running
    the solves one after another (deterministic kernels, no shared state)."""
    if concurrency <= 1 or len(jobs) <= 1 or device is None or torch.device(device).type != "cuda":
        return [dict(solve_one(j)) for j in jobs]
    from concurrent.futures import ThreadPoolExecutor
    dev = torch.device(device)

    def task(j):
        torch.cuda.set_device(dev)
        s = torch.cuda.Stream(dev)
        with torch.cuda.stream(s):
            rep = dict(solve_one(j))
        s.synchronize()
        return rep

    from . import _lib
    with _lib.concurrent_problems(), ThreadPoolExecutor(max_workers=min(concurrency, len(jobs))) as ex:
        return list(ex.map(task, jobs))


def solve_rhs_sharded(n_rhs: int, rank: int, world: int, solve_one, group=None, concurrency: int = 1,
                      device=None):
    """Run solve_one(j) -> dict for this rank's RHS (``concurrency`` of them at
    a time on separate CUDA streams of ``device``), gather all reports on every
    rank (host objects), return (reports sorted by j, aggregate dict).
    Aggregate it/s = sum of iterations / max over ranks of the wall time."""
    t0 = time.perf_counter()
    jobs = rhs_assignment(n_rhs, world, rank)
    mine = _run_concurrently(jobs, solve_one, concurrency, device)
    for j, rep in zip(jobs, mine):
        rep["rhs"] = j
        rep["rank"] = rank
    wall = time.perf_counter() - t0
    if world > 1:
        allr = [None] * world
        dist.all_gather_object(allr, {"reports": mine, "wall": wall}, group=group)
    else:
        allr = [{"reports": mine, "wall": wall}]
    reports = sorted((r for a in allr for r in a["reports"]), key=lambda r: r["rhs"])
    max_wall = max(a["wall"] for a in allr)
    iters = sum(r.get("iterations", 0) for r in reports)
    agg = {"n_rhs": n_rhs, "world": world, "iterations": iters, "max_wall_s": max_wall,
           "it_per_s": iters / max_wall if max_wall > 0 else 0.0, "concurrency": concurrency}
    return reports, agg
