"""Benchmark of the B200 TT-sGMRES hot path (BASELINE.json metric).

Headline workload (BASELINE.json configs[2], "TT matvec + rounding"): one step
applies the d=32, n=128, op-rank-3 anisotropic convection-diffusion TT
operator to a rank-64 Gaussian TT (tt_matvec, output rank 192) and rounds the
result with randomize-then-orthogonalize at sketch rank l=80 followed by TT-SVD
truncation to rank 64.  value = (matvec + RTO-sweep FLOPs) / step time in
GFLOP/s (the truncation is timed but not counted).  The step is the public
tt_matvec_round_rto call; e2e runs it on pinned host cores (uploads and the
result download overlap the compute), inflight runs 2 / 4 independent problems
on separate streams.

The same line carries the rest of the BASELINE metric ("... & TT-sGMRES
iters/s"): ``solver`` (config 1, config 5 RHS 0: it/s and time to 1e-6, CPU
oracle / committed reference wall time beside them) and ``sharded`` (the two
workloads that partition over GPUs: config-4 Khatri-Rao rows
with an NCCL all-gather, config-5 right-hand sides j on rank j mod G).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--extras]

--gpus N without torchrun re-launches this script as N ranks under
torch.distributed.run (127.0.0.1); under torchrun the world size must equal
--gpus.  The config-3 headline runs as independent replicas on every rank
(the rounding chain does not shard -- "replicas only"): value is
the FLOPs of all ranks / the max-over-ranks device time.  --impl reference
times the CPU oracle (numpy restatement of the reference path, oracle/) on
the host cores for the same workload (rank 0 only).
"""

from __future__ import annotations

import os

if "OPENBLAS_NUM_THREADS" not in os.environ:  # CPU legs use every host core
    os.environ["OPENBLAS_NUM_THREADS"] = str(os.cpu_count() or 1)
    os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count() or 1))

import argparse
import json
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "randomized TT-round+matvec GFLOP/s (fp64)"
UNIT = "GFLOP/s"
WORKLOAD = ("config3: tt_matvec of the d=32 n=128 op-rank-3 convection-diffusion TT operator on a "
            "rank-64 Gaussian TT (-> rank 192), then randomize-then-orthogonalize rounding l=80 + "
            "TT-SVD truncation to rank 64")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--concurrency", type=int, default=8,
                   help="solver workload: independent RHS solved at once per GPU (one CUDA stream each)")
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--extras", action="store_true", help="also time configs 1, 2, 4 and 5")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--workload", default="cfg3", choices=["cfg3", "kr", "solver"],
                   help="cfg3 (headline, replicas), kr (config 4, rows sharded over ranks + all-gather), "
                        "solver (config 5, 8 right-hand sides sharded over ranks)")
    p.add_argument("--no-solver", action="store_true", help="skip the solver / sharded objects")
    p.add_argument("--launcher-selftest", action="store_true",
                   help="(tests) start the ranks exactly as --gpus N does, join a gloo group, print n_gpus")
    return p.parse_args()


# ---------------------------------------------------------------------------
# launcher: --gpus N starts N ranks itself when not already under torchrun

def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def launch_ranks(n):
    """Re-exec this script as ``n`` ranks under torch.distributed.run (one
    process per GPU, rendezvous on 127.0.0.1); returns the launcher's exit code."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__),
           *sys.argv[1:]]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")          # the communicator reports nranks on stderr
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("OMP_NUM_THREADS", str(max(1, (os.cpu_count() or 1) // n)))
    return subprocess.call(cmd, env=env)


def world_from_env(args):
    """World size / rank of this process; the world must equal --gpus."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch with "
                         f"torchrun --nproc-per-node {args.gpus} or without torchrun")
    return world, int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0"))


def launcher_selftest(args):
    import torch
    import torch.distributed as dist
    world, rank, _ = world_from_env(args)
    dist.init_process_group("gloo")
    t = torch.ones(1)
    dist.all_reduce(t)
    if rank == 0:
        print(json.dumps({"n_gpus": world, "all_reduce": float(t.item()), "backend": "gloo",
                          "launcher": "torch.distributed.run" if "TORCHELASTIC_RUN_ID" in os.environ else "env"}),
              flush=True)
    dist.destroy_process_group()
    return 0


def bench_config(C, flops, mv_flops, rto_fl, world):
    """The config object both arms print (identical keys and values for the same N)."""
    return {"workload": WORKLOAD, "parallelism": f"replicas x{world}" if world > 1 else "single",
            "flops_per_step": flops, "matvec_flops": mv_flops, "rto_sweep_flops": rto_fl,
            "dims": [int(C["dims"][0])] * len(C["dims"]), "x_rank": 64, "op_rank": 3, "ell": C["ell"],
            "max_rank": C["max_rank"], "rel_tol": C["rel_tol"],
            "l2": "inputs larger than L2 (matvec output 1.13 GB per step)"}


# ---------------------------------------------------------------------------
# clocks sampled during the timed region (B200_PROFILING.md recipe)

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for nm, v in zip(names, s[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------

def fp64_peak(torch, dev):
    """cuBLAS DGEMM 4096^3, best of 5 (the FP64 tensor-pipe roofline denominator;
    MEASURED_PEAKS.json carries no fp64 entry)."""
    n = 4096
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); a @ b; e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    return 2.0 * n ** 3 / (best * 1e-3) / 1e9


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def subspace_roofline(T, torch, dev, stream, z, r, calls_per_step=None, step_ms=None):
    """The step's largest kernel by time is the gap-certified subspace
    factorisation of the truncation (qr.cu trunc_subspace_kernel, one per core,
    a sequential chain): ONE CTA holds the l x l Gram and every l x r iterate in
    shared memory; 12 DMMA products and two blocked Cholesky factorisations with
    explicit inverses per pass.  Time it live on the Gram of the step's own last
    unfolding and report its algorithmic FLOPs against the DMMA peak of the one
    SM it occupies; the bound is that SM's DMMA issue rate plus the 2 x r pivot
    chain of the Cholesky factorisations."""
    from paper_2409_09471_b200 import _lib
    lib = _lib.load()
    c = z.cores[-1]
    l = int(c.shape[0])
    cm = c.reshape(l, -1)
    G = (cm @ cm.T).contiguous()
    F = torch.empty((l, l), dtype=torch.float64, device=dev)
    Mt = torch.empty((l, l), dtype=torch.float64, device=dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    info = torch.zeros(4, dtype=torch.float64, device=dev)
    call = lambda: _lib.check(lib.ttk_debug_trunc_subspace(l, r, G.data_ptr(), F.data_ptr(), Mt.data_ptr(),
                                                           flag.data_ptr(), info.data_ptr(), None,
                                                           _lib.stream_ptr(dev)))
    call()
    torch.cuda.synchronize()
    if len(z.cores) > 2:
        # the typical instance is an interior core (flat kept spectrum, one pass); the two
        # end cores carry the whole spectrum (kappa ~26) and take two passes.  Interior
        # unfolding: C_{d-2} x_3 F, as the truncation forms it
        p = z.cores[-2]
        cm = (p.reshape(-1, l) @ F[:, :r]).reshape(int(p.shape[0]), -1)
        l = int(p.shape[0])
        G = (cm @ cm.T).contiguous()
        call()
        torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(5):
        call()
    b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    passes = int(info[2].item())
    # products (M, N, K) of the first pass (DESIGN 2.2): 4 of r x r x l, 4 of l x r x r, 4 of l x r x l;
    # a further pass adds 2 + 3 + 3 of them; two (one) Cholesky + triangular inverse of order r per pass
    mac = lambda n_rrl, n_lrr, n_lrl: n_rrl * r * r * l + n_lrr * l * r * r + n_lrl * l * r * l
    flops = 2.0 * (mac(4, 4, 4) + (passes - 1) * mac(3, 3, 3)) + (passes + 1) * (2.0 * r ** 3 / 3.0)
    sm_peak = 37.1e3 / 148  # GFLOP/s of one SM: measured DMMA issue peak / SM count (profiles/fp64_peak_r01.log)
    ach = flops / (ms * 1e-3) / 1e9
    out = {"kernel": "trunc_subspace_kernel (one CTA, %dx%d Gram -> rank %d, %d pass%s; second core from the right of the step)"
                     % (l, l, r, passes, "" if passes == 1 else "es"),
           "ms": ms, "passes": passes, "certified": int(flag.item()), "angle_bound": float(info[0].item()),
           "bound": "one SM: DMMA issue rate of the l x r products + the sequential pivot chain of "
                    "two r x r Cholesky factorisations per pass",
           "algorithmic_flops": flops, "achieved_gflops": ach, "sms": 1, "peak_gflops_of_its_sms": sm_peak,
           "frac_of_its_sms": ach / sm_peak}
    if calls_per_step and step_ms:
        out["share_of_step_est"] = calls_per_step * ms / step_ms
        out["share_basis"] = "%d calls/step x this single-call time / ms_per_step" % calls_per_step
    return out


def cfg3_flops(C):
    from paper_2409_09471_b200.configs import matvec_flops
    from paper_2409_09471_b200.rto import rto_flops, rto_ranks
    xr = [1] + [c.shape[2] for c in C["x"]]
    mv = matvec_flops(C["op"], xr)
    yr = [1] + [c.shape[2] * g.shape[3] for c, g in zip(C["x"], C["op"])]
    ls = rto_ranks(C["dims"], yr, C["ell"])
    return mv, rto_flops(C["dims"], yr, ls)


def cpu_oracle_step(C):
    import oracle as O
    y = O.matvec(C["op"], C["x"])
    return O.rto_round(y, C["drm"], C["rel_tol"], C["max_rank"])


def cpu_baseline(C, flops, budget_s=20.0):
    """The oracle port on the host cores; bounded sample = whole steps until
    ~budget_s of CPU work (at least one)."""
    t0 = time.perf_counter()
    cpu_oracle_step(C)  # warm-up (BLAS thread pool, page faults)
    t_warm = time.perf_counter() - t0
    reps = max(1, min(3, int(budget_s / max(t_warm, 1e-3))))
    ts, out = [], None
    for _ in range(reps):
        t0 = time.perf_counter()
        out = cpu_oracle_step(C)
        ts.append(time.perf_counter() - t0)
    t = float(np.median(ts))
    return {"value": flops / t / 1e9, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
            "sample": f"{reps} full config-3 steps after 1 warm-up (median {t:.2f} s/step); numpy "
                      f"restatement oracle/ttoracle.py (matvec + rto_round), OpenBLAS threads = "
                      f"{os.environ.get('OPENBLAS_NUM_THREADS')}",
            "s_per_step": t}, out


# ---------------------------------------------------------------------------

def run_reference(args):
    """The reference arm: the CPU oracle (numpy + OpenBLAS on every host core)
    on the same config-3 workload; under torchrun only rank 0 runs it."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from paper_2409_09471_b200 import configs
    C = configs.config3()
    mv, rto = cfg3_flops(C)
    flops = mv + rto
    for _ in range(args.warmup):
        cpu_oracle_step(C)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        cpu_oracle_step(C)
        ts.append(time.perf_counter() - t0)
    tot = sum(ts)
    value = flops * args.steps / tot / 1e9
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": bench_config(C, flops, mv, rto, world),
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                             "sample": f"{args.steps} full config-3 steps (numpy restatement of the "
                                       f"reference path, oracle/ttoracle.py; the Python reference "
                                       f"itself is not on the GPU box)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_b200(args):
    import torch
    import torch.distributed as dist
    import paper_2409_09471_b200 as T
    from paper_2409_09471_b200 import _lib, configs

    world, rank, local = world_from_env(args)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    lib = _lib.load()

    C = configs.config3()
    mv_flops, rto_fl = cfg3_flops(C)
    flops = mv_flops + rto_fl
    spec = T.RoundSpec(C["rel_tol"], C["max_rank"])
    op = T.TTOperator(C["op"], device=dev)
    x = T.TTVector(C["x"], device=dev)
    drm = [torch.as_tensor(g, device=dev) for g in C["drm"]]

    # the step through the public API: tt_matvec_round_rto pipelines the same
    # three calls (per-chunk matvec overlapping the event-gated RTO right sweep);
    # BENCH_UNFUSED=1 times tt_matvec -> rto_sweeps -> tt_truncate_left_orth
    unfused = os.environ.get("BENCH_UNFUSED") == "1"

    def step(op, x):
        if unfused:
            y = T.tt_matvec(op, x)
            return T.tt_truncate_left_orth(T.rto_sweeps(y, drm), spec)
        return T.tt_matvec_round_rto(op, x, spec, drm, device=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    # ---- device-resident timing (value) ----
    for _ in range(max(args.warmup, 3)):
        out = step(op, x)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    n0 = lib.ttk_launch_count()
    stream = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        e0.record(stream)
        for _ in range(args.steps):
            out = step(op, x)
        e1.record(stream)
        torch.cuda.synchronize()
    launches = (lib.ttk_launch_count() - n0) // args.steps
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    barrier()

    # ---- phase breakdown of one step (device events) ----
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record(stream)
    y = T.tt_matvec(op, x)
    ev[1].record(stream)
    z = T.rto_sweeps(y, drm)
    ev[2].record(stream)
    T.tt_truncate_left_orth(z, spec)
    ev[3].record(stream)
    torch.cuda.synchronize()
    phases = {"matvec_ms": ev[0].elapsed_time(ev[1]), "rto_sweeps_ms": ev[1].elapsed_time(ev[2]),
              "truncation_ms": ev[2].elapsed_time(ev[3])}

    # ---- dominant kernel roofline: the matvec grouped DMMA GEMM (one launch) ----
    reps = 5
    ybuf = [c for c in y.cores]  # reuse the output cores: time the launch only
    T.tt_matvec(op, x, out=ybuf)
    torch.cuda.synchronize()
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k0.record(stream)
    for _ in range(reps):
        T.tt_matvec(op, x, out=ybuf)
    k1.record(stream)
    torch.cuda.synchronize()
    mv_ms = k0.elapsed_time(k1) / reps
    peak = fp64_peak(torch, dev)
    achieved = mv_flops / (mv_ms * 1e-3) / 1e12
    # dram__bytes_read.sum + dram__bytes_write.sum of this launch from the committed
    # ncu --set full capture (profiles/r01_matvec_traffic.json)
    traffic, traffic_src = None, "none"
    tpath = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r01_matvec_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            tj = json.load(f)
        traffic, traffic_src = tj.get("traffic_bytes"), "ncu --set full, " + tj.get("source", tpath)
    roofline = {"bound": "tensor", "kernel": "gemm_group_kernel<64,32> (tt_matvec, 1 grouped launch/step)",
                "achieved": achieved, "peak": peak / 1e3, "unit": "TFLOP/s", "frac": achieved / (peak / 1e3),
                "peak_source": "live cuBLAS DGEMM 4096^3 (fp64 tensor pipe; MEASURED_PEAKS.json has no "
                               "fp64 entry; DMMA issue peak measured 37.1 TF/s, profiles/fp64_peak_r01.log)",
                "traffic": traffic, "traffic_source": traffic_src,
                "algorithmic_flops": mv_flops,
                "algorithmic_bytes": 8.0 * sum(c.numel() for c in y.cores)}
    roofline["dominant_kernel"] = subspace_roofline(T, torch, dev, stream, z, int(C["max_rank"]),
                                                    calls_per_step=len(C["x"]) - 1, step_ms=ms)

    # ---- end-to-end through the public API with host buffers ----
    host_op = [torch.as_tensor(g).pin_memory() for g in C["op"]]
    host_x = [torch.as_tensor(c).pin_memory() for c in C["x"]]
    h2d = sum(t.numel() * 8 for t in host_op + host_x)
    res_host = None

    def e2e_step():
        if unfused:
            a = T.TTOperator([t.to(dev, non_blocking=True) for t in host_op], device=dev)
            v = T.TTVector([t.to(dev, non_blocking=True) for t in host_x], device=dev)
            r = step(a, v)
            return [c.to("cpu", non_blocking=True) for c in r.cores]
        # host (pinned) cores in, host cores out: uploads, contraction, rounding
        # and the result download overlap inside the call
        r = T.tt_matvec_round_rto(T.TTOperator(host_op), T.TTVector(host_x), spec, drm, device=dev)
        return list(r.cores)

    for _ in range(2):
        res_host = e2e_step()
    torch.cuda.synchronize()
    barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for _ in range(args.steps):
        res_host = e2e_step()
    f1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = f0.elapsed_time(f1) / args.steps
    if world > 1:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    d2h = sum(c.numel() * 8 for c in res_host)
    # the host-pipeline result of the last timed step against the device-resident result
    # (same tensor; its chunked right sweep runs on the cp.async GEMM, DESIGN 6.2)
    import oracle as _O
    e2e_rel = float(_O.rel_diff([h.cpu().numpy() for h in res_host], [g.cpu().numpy() for g in out.cores]))

    # ---- independent problems in flight (serving-loop throughput; reported beside
    # the single-problem headline, which stays the latency-bound chain) ----
    def inflight(n, steps):
        streams = [torch.cuda.Stream(dev) for _ in range(n)]
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ends = [torch.cuda.Event() for _ in range(n)]

        last = [None] * n

        def worker(i, k):
            torch.cuda.set_device(dev)
            streams[i].wait_event(g0)
            with torch.cuda.stream(streams[i]):
                for _ in range(k):
                    last[i] = step(op, x)
            ends[i].record(streams[i])

        def run(k):
            g0.record(stream)
            ths = [threading.Thread(target=worker, args=(i, k)) for i in range(n)]
            [t.start() for t in ths]
            [t.join() for t in ths]
            for e in ends:
                stream.wait_event(e)
            g1.record(stream)
            torch.cuda.synchronize()
            return g0.elapsed_time(g1)
        with _lib.concurrent_problems():  # several problems in flight: cp.async GEMMs (DESIGN 6.2)
            run(1)  # warm-up: per-stream workspaces, per-thread side streams
            ms_all = run(steps)
        # every problem's last result is the lone run's tensor (||a - b|| through dot
        # products: cancellation floor ~1e-8; DESIGN 6.2)
        nref = float(T.tt_norm(out))
        dev_rel = [float(T.tt_norm(T.tt_add(r, T.tt_scale(out, -1.0)))) / nref for r in last]
        return {"problems_in_flight": n, "steps_each": steps, "value": flops * n * steps / (ms_all * 1e-3) / 1e9,
                "verified": bool(max(dev_rel) <= 1e-6), "max_rel_diff_vs_single": max(dev_rel),
                "unit": UNIT, "ms_per_problem_per_stream": ms_all / steps}
    inflight_res = None
    if world == 1:
        try:
            inflight_res = {str(n): inflight(n, max(2, args.steps // 2)) for n in (2, 4)}
        except Exception as exc:  # the headline must not depend on the extra measurement
            inflight_res = {"error": repr(exc)[:200]}

    peak_tf = peak / 1e3
    step_tf = flops / (ms * 1e-3) / 1e12
    roofline["step_frac"] = step_tf / peak_tf
    roofline["step_achieved"] = step_tf
    dk = roofline["dominant_kernel"]
    dk["chip_frac"] = dk["achieved_gflops"] / 1e3 / peak_tf
    roofline["note"] = ("frac/achieved: the matvec GEMM (the one FLOP-bound kernel, one launch per step); "
                        "step_frac: whole step (matvec + RTO sweep FLOPs / step time) vs the same fp64 peak; "
                        "dominant_kernel: the truncation's subspace factorisation (largest single kernel of the step), "
                        "chip_frac against the whole chip's fp64 peak")

    line = {"metric": METRIC, "value": flops * world / (ms * 1e-3) / 1e9, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": bench_config(C, flops, mv_flops, rto_fl, world),
            "out_ranks_max": max(out.ranks),
            "roofline": roofline,
            "e2e": {"value": flops * world / (e2e_ms * 1e-3) / 1e9, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms, "rel_diff_vs_device_result": e2e_rel,
                    "note": "h2d = operator + vector cores uploaded every step; the Gaussian TT-DRM of the "
                            "rounding (197 MB, a per-solve constant drawn once) stays resident on the device"},
            "gpu_launches": int(launches),
            "inflight": inflight_res,
            "clocks": clocks.summary(),
            "breakdown": phases}

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb, cpu_out = cpu_baseline(C, flops)
        line["cpu_baseline"] = cb
        import oracle as O
        line["parity"] = {"rel_diff_vs_oracle": O.rel_diff([c.cpu().numpy() for c in out.cores], cpu_out),
                          "ranks_equal": list(out.ranks) == [1] + [c.shape[2] for c in cpu_out]}
    del y, z, ybuf, out
    torch.cuda.empty_cache()
    if not args.no_solver:
        if rank == 0:
            try:
                line["solver"] = solver_metrics(T, torch, dev, cpu=(world == 1 and not args.no_cpu_baseline))
            except Exception as exc:  # the headline must not depend on the extra measurement
                line["solver"] = {"error": repr(exc)[:300]}
        barrier()
        line["sharded"] = {"kr": sharded_kr(args, T, torch, dev, world, rank, local, peak_tf),
                           "solver": sharded_solver(args, T, torch, dev, world, rank, local)}
    if args.extras and rank == 0:
        line["extras"] = run_extras(T, torch, dev)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


# ---------------------------------------------------------------------------
# TT-sGMRES iterations/s (the second half of the BASELINE metric)

def _solver_inputs(T, torch, dev, C, rounding):
    cfg = T.SolverConfig(**C["cfg"], zero_rel=None, rounding=rounding)
    a = T.TTOperator(C["op"], device=dev)
    b = T.TTVector(C["b"], device=dev)
    s = T.kr_sketch_new(C["dims"], cfg.sketch_rows, seed=C["sketch_seed"], device=dev)
    frame = T.make_solver_frame(b, cfg, seed=C["frame_seed"])
    return cfg, a, b, s, frame


def _timed_solve(T, torch, dev, C, rounding):
    """One untimed warm-up solve capped at 4 iterations (lazy kernel loading,
    grow-only workspaces), then the timed solve; wall clock around the whole
    solve (it synchronises the host every iteration) and the phase split from
    the solver's CUDA-event timer."""
    cfg, a, b, s, frame = _solver_inputs(T, torch, dev, C, rounding)
    warm = T.SolverConfig(**{**C["cfg"], "maxit": 4}, zero_rel=None, rounding=rounding)
    T.tt_sgmres(a, b, None, warm, s, T.make_solver_frame(b, warm, seed=C["frame_seed"]))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, rep = T.tt_sgmres(a, b, None, cfg, s, frame)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    return {"rounding": rounding, "iterations": rep.iterations, "converged": rep.converged, "wall_s": wall,
            "it_per_s": rep.iterations / wall, "final_res_sketched": rep.res_sketched[-1],
            "time_to_1e-6_s": rep.time_to_tol.get(1e-6), "peak_rank": rep.peak_rank,
            "phase_s": rep.phase_totals()}


def _fixture(name):
    try:
        return np.load(os.path.join(ROOT, "tests", "golden", name), allow_pickle=False)
    except Exception:
        return None


def solver_metrics(T, torch, dev, cpu=True):
    """Config 1 (40 iterations) and config 5 RHS 0 on one GPU, both rounding
    modes; the CPU oracle's config-1 solve (randomized rounding, same inputs)
    timed beside it, and the committed reference run's config-5 wall time
    (tests/golden/solver_cfg5.npz, measured in the build container) quoted."""
    from paper_2409_09471_b200 import configs
    out = {"unit": "it/s", "timing": "host wall clock around tt_sgmres after an untimed 4-iteration warm-up"}
    C1 = configs.config1()
    out["config1"] = {"rto": _timed_solve(T, torch, dev, C1, "rto"), "svd": _timed_solve(T, torch, dev, C1, "svd")}
    if cpu:
        import oracle as O
        g = out["config1"]["rto"]
        cfg = {**C1["cfg"], "zero_rel": None, "oversampling": 20}
        drm = [x.cpu().numpy() for x in T.solver_rto_drm(C1["dims"], T.SolverConfig(**C1["cfg"], zero_rel=None,
                                                                                     rounding="rto"),
                                                         device=dev).cores]
        f = O.kr_factors_new(C1["dims"], cfg["sketch_rows"], seed=C1["sketch_seed"])
        t0 = time.perf_counter()
        _, orep = O.sgmres(C1["op"], C1["b"], cfg, f, frame=O.solver_frame(C1["b"], cfg, seed=C1["frame_seed"]),
                           rounding="rto", rto_drm=drm)
        wall = time.perf_counter() - t0
        out["config1"]["cpu_baseline"] = {
            "value": orep["iterations"] / wall, "unit": "it/s", "cores": os.cpu_count(), "kind": "port",
            "sample": f"one full config-1 solve, randomized rounding ({orep['iterations']} iterations, "
                      f"{wall:.2f} s), oracle/ttoracle.py sgmres",
            "same_history": orep["iterations"] == g["iterations"]}
    C5 = configs.config5(0)
    out["config5_rhs0"] = {"rto": _timed_solve(T, torch, dev, C5, "rto"), "svd": _timed_solve(T, torch, dev, C5, "svd")}
    z = _fixture("solver_cfg5.npz")
    if z is not None:
        it = int(z["cfg5_0_iters"])
        res = z["cfg5_0_res"]
        cum = np.cumsum(z["cfg5_0_iter_s"])
        hit = [i for i, r in enumerate(res) if r <= 1e-6]
        out["config5_rhs0"]["reference_run"] = {
            "kind": "reference (recorded)", "iterations": it, "wall_s": float(z["cfg5_0_wall"]),
            "it_per_s": it / float(z["cfg5_0_wall"]), "cores": 8,
            "time_to_1e-6_s": float(cum[hit[0]]) if hit else None,
            "sample": "the reference ttkrylov tt_sgmres (TT-SVD rounding, Q1 bypassed) timed in the build "
                      "container (8 cores, OpenBLAS) when the committed fixture was made -- not this box"}
    return out


# ---------------------------------------------------------------------------
# the two workloads that shard over GPUs

def sharded_kr(args, T, torch, dev, world, rank, local, peak_tf):
    """Config 4: s=512 Khatri-Rao rows split over the ranks, all 64 vectors
    replicated (drawn on rank 0, NCCL broadcast), one NCCL all-gather of the
    (64 x s/G) blocks per step; value = batch FLOPs / max-over-ranks time."""
    import torch.distributed as dist
    from paper_2409_09471_b200 import _lib, configs
    from paper_2409_09471_b200.parallel import kr_apply_sharded, row_partition
    d, n, r, s, B = 20, 64, 100, 512, 64
    full = [1] + [r] * (d - 1) + [1]
    if rank == 0:
        C = configs.config4()
        fac = [torch.as_tensor(f, device=dev) for f in C["factors"]]
        vecs = [[torch.as_tensor(c, device=dev) for c in v] for v in C["vecs"]]
        del C
    else:
        fac = [torch.empty((s, n), dtype=torch.float64, device=dev) for _ in range(d)]
        vecs = [[torch.empty((full[k], n, full[k + 1]), dtype=torch.float64, device=dev) for k in range(d)]
                for _ in range(B)]
    if world > 1:
        for t in fac + [c for v in vecs for c in v]:
            dist.broadcast(t, 0)
    sk = T.KhatriRaoSketch(fac, device=dev)
    vs = [T.TTVector(v, device=dev) for v in vecs]
    flops = sum(2.0 * s * n * r0 * r1 for r0, r1 in zip(full[:-1], full[1:])) * B
    lo, hi = row_partition(s, world)[rank]
    lib = _lib.load()
    for _ in range(3):
        out = kr_apply_sharded(sk, vs, rank, world)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    st = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = max(args.steps // 2, 3)
    n0 = lib.ttk_launch_count()
    e0.record(st)
    for _ in range(steps):
        out = kr_apply_sharded(sk, vs, rank, world)
    e1.record(st)
    torch.cuda.synchronize()
    launches = (lib.ttk_launch_count() - n0) // steps
    ms = _max_over_ranks(torch, dev, world, e0.elapsed_time(e1) / steps)
    # the kernel alone (this rank's rows, no gather)
    k0.record(st)
    for _ in range(steps):
        T.kr_apply_rows(sk, vs, lo, hi)
    k1.record(st)
    torch.cuda.synchronize()
    kms = _max_over_ranks(torch, dev, world, k0.elapsed_time(k1) / steps)
    res = {"metric": "Khatri-Rao sketch GFLOP/s (fp64), config 4", "value": flops / (ms * 1e-3) / 1e9,
           "unit": UNIT, "n_gpus": world, "scaling": "strong", "ms_per_step": ms, "steps": steps,
           "config": {"workload": "config4: s=512 rows, 64 TTs d=20 n=64 r=100, N(0,1/n) factors; rows split "
                                  "over ranks, NCCL all-gather of the row blocks", "rows_per_rank": hi - lo,
                      "flops_per_step": flops},
           "gpu_launches": int(launches),
           "roofline": {"bound": "tensor", "kernel": "kr_fused_kernel (this rank's rows, all 64 vectors)",
                        "achieved": flops / world / (kms * 1e-3) / 1e12, "peak": peak_tf, "unit": "TFLOP/s",
                        "frac": flops / world / (kms * 1e-3) / 1e12 / peak_tf, "kernel_ms": kms,
                        "traffic": None}}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle as O
        C1 = configs.config4(nvec=1)
        t0 = time.perf_counter()
        want = O.kr_apply(C1["factors"], C1["vecs"][0])
        t = time.perf_counter() - t0
        got = out[0].cpu().numpy()
        res["cpu_baseline"] = {"value": flops / B / t / 1e9, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                               "sample": f"oracle kr_apply of vector 0 (all 512 rows, {t:.2f} s)"}
        res["parity"] = {"vector0_rel_diff": float(np.linalg.norm(got - want) / np.linalg.norm(want))}
    del vs, vecs, fac, sk, out
    torch.cuda.empty_cache()
    return res


def sharded_solver(args, T, torch, dev, world, rank, local):
    """Config 5: 8 right-hand sides, RHS j on rank j mod G (no device
    collective, reports gathered on the host), each rank's RHS solved
    concurrently on their own CUDA streams; randomized rounding."""
    import torch.distributed as dist
    from paper_2409_09471_b200 import configs
    from paper_2409_09471_b200.parallel import rhs_assignment, solve_rhs_sharded
    n_rhs = 8
    prepared = {}
    for j in rhs_assignment(n_rhs, world, rank):
        prepared[j] = _solver_inputs(T, torch, dev, configs.config5(j), "rto")
    torch.cuda.synchronize()

    def warm_one(j):
        cfg, a, b, sk, frame = prepared[j]
        w = T.SolverConfig(**{**configs.config5(j)["cfg"], "maxit": 4}, zero_rel=None, rounding="rto")
        T.tt_sgmres(a, b, None, w, sk, frame)
        torch.cuda.current_stream(dev).synchronize()
        return {"iterations": 0}

    def solve_one(j):
        cfg, a, b, sk, frame = prepared[j]
        t0 = time.perf_counter()
        _, rep = T.tt_sgmres(a, b, None, cfg, sk, frame)
        torch.cuda.current_stream(dev).synchronize()
        return {"iterations": rep.iterations, "converged": rep.converged, "wall_s": time.perf_counter() - t0,
                "res_sketched": rep.res_sketched[-1], "peak_rank": rep.peak_rank,
                "time_to_1e-6_s": rep.time_to_tol.get(1e-6)}
    solve_rhs_sharded(n_rhs, rank, world, warm_one, concurrency=args.concurrency, device=dev)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    reports, agg = solve_rhs_sharded(n_rhs, rank, world, solve_one, concurrency=args.concurrency, device=dev)
    ttt = [r["time_to_1e-6_s"] for r in reports if r.get("time_to_1e-6_s") is not None]
    return {"metric": "TT-sGMRES iterations/s (fp64), config 5, 8 RHS", "value": agg["it_per_s"], "unit": "it/s",
            "n_gpus": world, "scaling": "strong", "iterations": agg["iterations"], "max_wall_s": agg["max_wall_s"],
            "time_to_1e-6_s_max": max(ttt) if ttt else None,
            "config": {"workload": "config5: d=50 n=256, ell=3, s=120, maxit=60, tol=1e-8, cap 100, RTO rounding; "
                                   "RHS j on rank j mod G, a rank's RHS on concurrent CUDA streams",
                       "concurrency": args.concurrency},
            "reports": [{k: r[k] for k in ("rhs", "rank", "iterations", "converged", "wall_s", "time_to_1e-6_s")}
                        for r in reports]}


def run_extras(T, torch, dev):
    """Configs 2 and 4 (kernel GFLOP/s) and the solver configs 1 and 5 (it/s)."""
    from paper_2409_09471_b200 import configs
    from paper_2409_09471_b200.rto import rto_flops, rto_ranks
    out = {}
    st = torch.cuda.current_stream(dev)

    def timed(fn, reps=3):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(reps):
            fn()
        b.record(st)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps
    # config 2
    C2 = configs.config2()
    x2 = T.TTVector(C2["x"], device=dev)
    drm2 = [torch.as_tensor(g, device=dev) for g in C2["drm"]]
    ls = rto_ranks(C2["dims"], list(x2.ranks), C2["ell"])
    f2 = rto_flops(C2["dims"], list(x2.ranks), ls)
    ms_sw = timed(lambda: T.rto_sweeps(x2, drm2))
    ms_all = timed(lambda: T.tt_truncate_left_orth(T.rto_sweeps(x2, drm2), T.RoundSpec(0.0, 40)))
    out["config2_rto"] = {"gflop": f2 / 1e9, "sweeps_ms": ms_sw, "sweeps_gflops": f2 / ms_sw / 1e6,
                          "with_truncation_ms": ms_all}
    # config 4
    C4 = configs.config4()
    sk = T.KhatriRaoSketch(C4["factors"], device=dev)
    vs = [T.TTVector(v, device=dev) for v in C4["vecs"]]
    f4 = sum(configs.kr_flops(C4["rows"], C4["dims"], list(v.ranks)) for v in vs)
    ms4 = timed(lambda: T.kr_apply_batch(sk, vs), reps=2)
    out["config4_kr"] = {"gflop": f4 / 1e9, "ms": ms4, "gflops": f4 / ms4 / 1e6}
    del vs, sk
    # solvers
    for name, builder in (("config1_sgmres_rto", configs.config1), ("config5_sgmres_rto", configs.config5)):
        C = builder()
        cfg = T.SolverConfig(**C["cfg"], zero_rel=None, rounding="rto")
        a = T.TTOperator(C["op"], device=dev)
        b = T.TTVector(C["b"], device=dev)
        s = T.kr_sketch_new(C["dims"], cfg.sketch_rows, seed=C["sketch_seed"], device=dev)
        frame = T.make_solver_frame(b, cfg, seed=C["frame_seed"])
        # untimed warm-up solve: lazy module loading of every kernel the solve
        # launches, grow-only workspaces, pinned scratch, side streams
        T.tt_sgmres(a, b, None, T.SolverConfig(**{**C["cfg"], "maxit": 4}, zero_rel=None, rounding="rto"), s,
                    T.make_solver_frame(b, cfg, seed=C["frame_seed"]))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, rep = T.tt_sgmres(a, b, None, cfg, s, frame)
        wall = time.perf_counter() - t0
        out[name] = {"iterations": rep.iterations, "converged": rep.converged, "wall_s": wall,
                     "it_per_s": rep.iterations / wall, "final_res_sketched": rep.res_sketched[-1],
                     "peak_rank": rep.peak_rank, "time_to_1e-6_s": rep.time_to_tol.get(1e-6),
                     "phase_s": rep.phase_totals()}
    return out


def _dist_setup(args):
    import torch
    import torch.distributed as dist
    world, rank, local = world_from_env(args)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if world > 1 and not dist.is_initialized():
        dist.init_process_group("nccl", device_id=dev)
    return world, rank, local, dev


def _max_over_ranks(torch, dev, world, v):
    if world == 1:
        return v
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_kr(args):
    """Config 4: 64 TTs (d=20, n=64, r=100) sketched with s=512 Khatri-Rao rows,
    rows sharded over the ranks, NCCL all-gather of the row blocks."""
    import torch
    import torch.distributed as dist
    import paper_2409_09471_b200 as T
    from paper_2409_09471_b200 import _lib, configs
    from paper_2409_09471_b200.parallel import kr_apply_sharded, row_partition
    world, rank, local, dev = _dist_setup(args)
    lib = _lib.load()
    C = configs.config4()
    sk = T.KhatriRaoSketch(C["factors"], device=dev)
    vs = [T.TTVector(v, device=dev) for v in C["vecs"]]
    flops_total = sum(configs.kr_flops(C["rows"], C["dims"], list(v.ranks)) for v in vs)
    lo, hi = row_partition(C["rows"], world)[rank]
    for _ in range(max(args.warmup, 3)):
        out = kr_apply_sharded(sk, vs, rank, world)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n0 = lib.ttk_launch_count()
    with ClockSampler(local) as clocks:
        e0.record(st)
        for _ in range(args.steps):
            out = kr_apply_sharded(sk, vs, rank, world)
        e1.record(st)
        torch.cuda.synchronize()
    ms = _max_over_ranks(torch, dev, world, e0.elapsed_time(e1) / args.steps)
    launches = (lib.ttk_launch_count() - n0) // args.steps
    line = {"metric": "Khatri-Rao sketch GFLOP/s (fp64), config 4", "value": flops_total / (ms * 1e-3) / 1e9,
            "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": "config4: s=512 rows, 64 TTs d=20 n=64 r=100; rows sharded, NCCL all-gather",
                       "rows_per_rank": hi - lo, "flops_per_step": flops_total},
            "gpu_launches": int(launches), "clocks": clocks.summary()}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_solver(args):
    """Config 5: 8 right-hand sides of the d=50, n=256 anisotropic Laplacian,
    RHS j on rank j mod G (no device collective), randomized rounding."""
    import torch
    import torch.distributed as dist
    import paper_2409_09471_b200 as T
    from paper_2409_09471_b200 import configs
    from paper_2409_09471_b200.parallel import solve_rhs_sharded
    world, rank, local, dev = _dist_setup(args)
    from paper_2409_09471_b200.parallel import rhs_assignment
    n_rhs = 8

    def prepare(j):
        # inputs (operator, RHS, Khatri-Rao sketch, STTA frame) are set up before
        # the clock, as the reference's own benchmark builds them before solving
        C = configs.config5(j)
        cfg = T.SolverConfig(**C["cfg"], zero_rel=None, rounding="rto")
        a = T.TTOperator(C["op"], device=dev)
        b = T.TTVector(C["b"], device=dev)
        sk = T.kr_sketch_new(C["dims"], cfg.sketch_rows, seed=C["sketch_seed"], device=dev)
        frame = T.make_solver_frame(b, cfg, seed=C["frame_seed"])
        return a, b, sk, frame, cfg

    prepared = {j: prepare(j) for j in rhs_assignment(n_rhs, world, rank)}
    torch.cuda.synchronize()

    def solve_one(j):
        a, b, sk, frame, cfg = prepared[j]
        st = torch.cuda.current_stream(dev)
        t0 = time.perf_counter()
        _, rep = T.tt_sgmres(a, b, None, cfg, sk, frame)
        st.synchronize()
        wall = time.perf_counter() - t0
        return {"iterations": rep.iterations, "converged": rep.converged, "wall_s": wall,
                "res_sketched": rep.res_sketched[-1], "peak_rank": rep.peak_rank,
                "time_to_1e-6_s": rep.time_to_tol.get(1e-6)}
    # untimed warm-up: the same concurrent solve capped at 4 iterations (kernel
    # module loading, per-stream workspaces, per-thread side streams and pinned
    # scratch all initialised before the clock)
    def warm_one(j):
        a, b, sk, frame, cfg = prepared[j]
        T.tt_sgmres(a, b, None, T.SolverConfig(**{**configs.config5(j)["cfg"], "maxit": 4}, zero_rel=None,
                                               rounding="rto"), sk, frame)
        torch.cuda.current_stream(dev).synchronize()
        return {"iterations": 0, "converged": False, "wall_s": 0.0, "res_sketched": 0.0, "peak_rank": 0,
                "time_to_1e-6_s": None}
    solve_rhs_sharded(n_rhs, rank, world, warm_one, concurrency=args.concurrency, device=dev)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    with ClockSampler(local) as clocks:
        reports, agg = solve_rhs_sharded(n_rhs, rank, world, solve_one, concurrency=args.concurrency,
                                         device=dev)
    line = {"metric": "TT-sGMRES iterations/s (fp64), config 5, 8 RHS", "value": agg["it_per_s"],
            "unit": "it/s", "n_gpus": world, "steps": n_rhs, "warmup": 0,
            "ms_per_step": agg["max_wall_s"] * 1e3 / max(1, n_rhs), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "config5: d=50 n=256, ell=3, s=120, maxit=60, tol=1e-8, cap 100, RTO rounding; "
                                   "RHS j on rank j mod G; a rank's RHS solved concurrently on "
                                   f"{args.concurrency} CUDA streams; inputs set up before the clock",
                       "parallelism": f"rhs x{world}", "concurrency": args.concurrency},
            "reports": reports, "clocks": clocks.summary()}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return launch_ranks(args.gpus)
    if args.launcher_selftest:
        return launcher_selftest(args)
    if args.impl == "reference":
        return run_reference(args)
    if args.workload == "kr":
        return run_kr(args)
    if args.workload == "solver":
        return run_solver(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
