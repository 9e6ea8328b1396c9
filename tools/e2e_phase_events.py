"""Phase events inside the host-buffer pipeline of tt_matvec_round_rto (a copy
of rto._matvec_round_rto with events; diagnostics)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2409_09471_b200 as T
from paper_2409_09471_b200 import configs, _lib
from paper_2409_09471_b200.rto import _pipe_streams, _drm_block, TTVector, ShapeMismatch, tt_truncate_left_orth
dev = torch.device("cuda", 0)
C = configs.config3()
spec = T.RoundSpec(C["rel_tol"], C["max_rank"])
drm = [torch.as_tensor(g, device=dev) for g in C["drm"]]
oph = T.TTOperator([torch.as_tensor(g).pin_memory() for g in C["op"]])
xh = T.TTVector([torch.as_tensor(c).pin_memory() for c in C["x"]])
opd = T.TTOperator(C["op"], device=dev); xd = T.TTVector(C["x"], device=dev)

def prof_round(a, v, spec, drm, chunk, device, E):
    if a.col_dims != v.dims:
        raise ShapeMismatch(f"operator col_dims {a.col_dims} do not match {v.dims}")
    host = v.device.type == "cpu"
    if host != (a.op_cores[0].device.type == "cpu"):
        raise ValueError("operator and vector must both be in host memory or both on the device")
    if not host:
        _lib.require_cuda(v.cores[0], "TT vector")
    dev = (torch.device(device) if device is not None
           else (torch.device("cuda", torch.cuda.current_device()) if host else v.device))
    lib = _lib.load()
    d = v.d
    rho, r = list(a.ranks), list(v.ranks)
    m, n = list(a.row_dims), list(a.col_dims)
    cur = torch.cuda.current_stream(dev)
    E[0].record(cur)
    up, mvs = _pipe_streams(dev)
    if host:
        xs = [torch.empty(tuple(c.shape), dtype=torch.float64, device=dev) for c in v.cores]
        ops = [torch.empty(tuple(c.shape), dtype=torch.float64, device=dev) for c in a.op_cores]
        ev_up = [torch.cuda.Event() for _ in range(d)]
        up.wait_stream(cur)  # the buffers were allocated on `cur`
        with torch.cuda.stream(up):
            for k in reversed(range(d)):
                ops[k].copy_(a.op_cores[k], non_blocking=True)
                xs[k].copy_(v.cores[k], non_blocking=True)
                ev_up[k].record(up)
        for t in ops + xs:
            t.record_stream(up)
    else:
        xs, ops, ev_up = list(v.cores), list(a.op_cores), None
    yr = [r[k] * rho[k] for k in range(d + 1)]
    y = [torch.empty((yr[k], m[k], yr[k + 1]), dtype=torch.float64, device=dev) for k in range(d)]
    # the DRM block is drawn on `cur` before the matvec stream starts
    ls, G = _drm_block(m, yr, drm, dev)
    mvs.wait_stream(cur)
    rho_a, m_a, n_a, r_a = (_lib.int_array(x) for x in (rho, m, n, r))
    D_p, C_p, Y_p = _lib.ptr_array(ops), _lib.ptr_array(xs), _lib.ptr_array(y)
    ev_mv = [None] * d
    if chunk is None:
        chunk = 4 if host else d
    chunk = max(1, int(chunk))
    for k1 in range(d, 0, -chunk):
        k0 = max(0, k1 - chunk)
        if ev_up is not None:
            mvs.wait_event(ev_up[k0])  # uploads run right to left: core k0 lands last
        _lib.check(lib.ttk_matvec_range(d, rho_a, m_a, n_a, r_a, D_p, C_p, Y_p, k0, k1, mvs.cuda_stream))
        e = torch.cuda.Event()
        e.record(mvs)
        for k in range(k0, k1):
            ev_mv[k] = e
    E[1].record(mvs)
    # RTO sweeps on `cur`, each core awaited on its matvec chunk's event
    L = [1] + ls + [1]
    z = [torch.empty((L[k], m[k], L[k + 1]), dtype=torch.float64, device=dev) for k in range(d)]
    if d == 1:
        cur.wait_event(ev_mv[0])
        z[0].copy_(y[0])
    else:
        dims_a, yr_a, L_a = _lib.int_array(m), _lib.int_array(yr), _lib.int_array(L)
        ws = _lib.workspace(lib.ttk_rto_ws_bytes(d, dims_a, yr_a, L_a), dev)
        ready = (_lib.ctypes.c_void_p * d)(*[e.cuda_event for e in ev_mv])
        _lib.check(lib.ttk_rto_sweeps_ev(d, dims_a, yr_a, _lib.ptr_array(y), L_a, _lib.ptr_array(G),
                                         _lib.ptr_array(z), ws.data_ptr(), ws.numel(), ready, cur.cuda_stream))
    E[2].record(cur)
    for t in ops + xs + y:  # read on `mvs` / `cur`: keep the blocks until both are done
        t.record_stream(mvs)
    zt = TTVector(z)
    if not host:
        res = tt_truncate_left_orth(zt, spec)
        E[3].record(cur)
        return res
    # truncation with every final core streamed into pinned host memory
    dims_a, ranks_a = _lib.int_array(zt.dims), _lib.int_array(zt.ranks)
    outs = [torch.empty(max(c.numel(), c.shape[1]), dtype=torch.float64, device=dev) for c in z]
    hosts = [torch.empty(max(c.numel(), c.shape[1]), dtype=torch.float64, pin_memory=True) for c in z]
    out_ranks = (_lib.ctypes.c_int * (d + 1))()
    if d == 1:
        hosts[0].copy_(z[0].reshape(-1))
        return TTVector([hosts[0][: m[0]].view(1, m[0], 1)])
    ws = _lib.workspace(lib.ttk_tt_truncate_ws_bytes(d, dims_a, ranks_a), dev)
    _lib.check(lib.ttk_tt_truncate_host(d, dims_a, ranks_a, _lib.ptr_array(z), float(spec.rel_tol),
                                        int(spec.max_rank or 0), _lib.ptr_array(outs), out_ranks,
                                        _lib.ptr_array(hosts), ws.data_ptr(), ws.numel(), cur.cuda_stream))
    E[3].record(cur)
    rr = list(out_ranks)
    return TTVector([hosts[k][: rr[k] * m[k] * rr[k + 1]].view(rr[k], m[k], rr[k + 1]) for k in range(d)])



for name, (o, x) in (("device", (opd, xd)), ("host", (oph, xh))):
    for rep in range(3):
        E = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        torch.cuda.synchronize()
        prof_round(o, x, spec, drm, None, dev, E)
        torch.cuda.synchronize()
        print(name, "matvec done %.2f  rto done %.2f  trunc done %.2f ms" % (E[0].elapsed_time(E[1]), E[0].elapsed_time(E[2]), E[0].elapsed_time(E[3])), flush=True)
