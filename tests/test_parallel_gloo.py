"""World-size-2 gloo tests of the multi-GPU partitioning (run on CPU):
Khatri-Rao row sharding with the fixed-order all-gather, and RHS sharding."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2409_09471_b200.parallel import (gather_row_blocks, kr_apply_sharded, rhs_assignment,
                                            row_partition, solve_rhs_sharded)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_row_partition_covers_rows():
    for rows in (1, 7, 80, 512, 513):
        for world in (1, 2, 3, 4, 8):
            parts = row_partition(rows, world)
            assert parts[0][0] == 0 and parts[-1][1] == rows
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            widths = [hi - lo for lo, hi in parts]
            assert max(widths) - min(widths) <= 1


def test_rhs_assignment_partition():
    for world in (1, 2, 4, 8):
        got = sorted(j for r in range(world) for j in rhs_assignment(8, world, r))
        assert got == list(range(8))


class _Sketch:
    def __init__(self, factors):
        self.factors = factors
        self.rows = factors[0].shape[0]


def _worker(rank, world, port, q):
    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        import oracle as O
        rng = np.random.default_rng(0)
        dims = [4, 5, 3, 6]
        factors = [rng.normal(0, 1 / np.sqrt(n), size=(37, n)) for n in dims]
        vecs = [O.tt_random(dims, [3, 4, 2], seed=10 + i) for i in range(3)]
        sk = _Sketch(factors)

        def compute(lo, hi):  # CPU oracle stands in for the device kernel
            return torch.tensor(np.stack([O.kr_apply([f[lo:hi] for f in factors], v) for v in vecs]))

        full = kr_apply_sharded(sk, vecs, rank, world, compute=compute)
        want = np.stack([O.kr_apply(factors, v) for v in vecs])
        ok_kr = bool(np.array_equal(full.numpy(), want))

        def solve_one(j):
            return {"iterations": j + 1, "converged": True}

        reps, agg = solve_rhs_sharded(5, rank, world, solve_one)
        ok_rhs = [r["rhs"] for r in reps] == list(range(5)) and agg["iterations"] == 15
        ok_ranks = all(r["rank"] == r["rhs"] % world for r in reps)
        q.put((rank, ok_kr, ok_rhs and ok_ranks))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported through the queue
        q.put((rank, repr(e), False))


def test_sharded_paths_world2_gloo():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok_kr, ok_rhs in res:
        assert ok_kr is True, f"rank {rank}: {ok_kr}"
        assert ok_rhs, f"rank {rank} rhs sharding"


def _gather_worker(rank, world, port, q):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    parts = row_partition(11, world)
    lo, hi = parts[rank]
    block = torch.arange(lo, hi, dtype=torch.float64).repeat(2, 1)
    full = gather_row_blocks(block, parts)
    q.put(bool(torch.equal(full, torch.arange(11, dtype=torch.float64).repeat(2, 1))))
    dist.destroy_process_group()


def test_uneven_gather_world2_gloo():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(res)


def test_bench_launcher_spawns_world2():
    """`python bench.py --gpus 2` without torchrun starts 2 ranks itself
    (torch.distributed.run on 127.0.0.1); the ranks join one process group and
    rank 0 reports n_gpus == 2."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                          "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--launcher-selftest"],
                         capture_output=True, text=True, timeout=300, env=env, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    assert lines[0]["n_gpus"] == 2 and lines[0]["all_reduce"] == 2.0
    assert lines[0]["launcher"] == "torch.distributed.run"


def test_bench_refuses_world_mismatch():
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--launcher-selftest"],
                         capture_output=True, text=True, timeout=300, env=env, cwd=root)
    assert out.returncode != 0 and "WORLD_SIZE=1" in out.stderr
