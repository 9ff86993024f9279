"""Python binding of the C ABI (include/gwdp.h): argument marshalling only.

Every step of the hot path runs in libgwdp.so's CUDA kernels; torch provides device
memory and the stream.  Names follow the C ABI: ``grad`` -> gw_grad_dp,
``sinkhorn`` -> sinkhorn_solve, ``solve`` -> entropic_gw_solve / fgw_solve.
"""

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from . import _lib as L

__all__ = ["Context", "grad", "sinkhorn", "solve", "solve_host", "ugw_solve", "Result", "plan_buffer"]


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


def _vec(v, device):
    t = torch.as_tensor(v, dtype=torch.float64, device=device)
    return t.contiguous()


def _ld(m):
    return (m + 31) // 32 * 32


def plan_buffer(n, m, device=None, dtype=torch.float32):
    """An (n, m) view into an (n, ld) buffer with ld % 32 == 0 (the ABI needs ld % 4 == 0)."""
    buf = torch.empty((n, _ld(m)), dtype=dtype, device=device)
    return buf[:, :m]


_GW_DTYPE = {torch.float32: L.GW_F32, torch.float64: L.GW_F64}


def _check_mat(t, name, dtype=None):
    """Leading dimension of a 2-D row-major float32 / float64 (GW_F64) CUDA matrix; `dtype`: required type."""
    if t.dtype not in _GW_DTYPE or not t.is_cuda or t.dim() != 2 or t.stride(1) != 1:
        raise ValueError("%s must be a 2-D row-major float32 or float64 CUDA tensor" % name)
    if dtype is not None and t.dtype != dtype:
        raise ValueError("%s must be %s like the other matrices of the call" % (name, dtype))
    return t.stride(0)


class Context:
    """One gw_ctx per (device, stream[, comm]); owns the library workspace.  `comm` is a
    dist.Comm (multi-rank) or None."""

    _cache = {}

    def __init__(self, device=None, stream=None, comm=None):
        if comm is not None and hasattr(comm, "ptr"):
            self.comm = comm
            comm = comm.ptr
        self.lib = L.load()
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else torch.device(device).index or 0)
        self.device = dev
        s = torch.cuda.current_stream(dev) if stream is None else stream
        self.stream = s
        h = C.c_void_p()
        L.check(self.lib.gw_ctx_create(C.byref(h), dev.index, C.c_void_p(s.cuda_stream),
                                       C.c_void_p(comm) if comm else C.c_void_p(0)))
        self.h = h

    @classmethod
    def get(cls, device=None):
        dev = torch.cuda.current_device() if device is None else torch.device(device).index or 0
        key = (dev, torch.cuda.current_stream(dev).cuda_stream)
        if key not in cls._cache:
            cls._cache[key] = Context(dev)
        return cls._cache[key]

    def trim(self):
        L.check(self.lib.gw_ctx_trim(self.h))

    def close(self):
        if self.h:
            self.lib.gw_ctx_destroy(self.h)
            self.h = None


def _problem(x, y, p, q, n_local=None, row0=0, flags=0, k=1, grid2d=False, dtype=torch.float32):
    pr = L.gw_problem()
    if grid2d:  # x, y are the grid axes (GW_GRID2D): n = len(p) = len(x)^2
        if p.numel() != x.numel() ** 2 or q.numel() != y.numel() ** 2:
            raise ValueError("grid2d: len(p) must be len(x)**2 and len(q) len(y)**2")
        flags |= L.GW_GRID2D
        pr.n, pr.m = p.numel(), q.numel()
    else:
        pr.n, pr.m = x.numel(), y.numel()
    pr.row0 = row0
    pr.n_local = pr.n if n_local is None else n_local
    pr.x, pr.y, pr.p, pr.q = x.data_ptr(), y.data_ptr(), p.data_ptr(), q.data_ptr()
    pr.k, pr.loss, pr.dtype, pr.flags = int(k), L.GW_LOSS_SQUARE, _GW_DTYPE[dtype], flags
    return pr


def grad(x, y, p, q, T, out=None, validate=True, ctx=None, row0=0, k=1, grid2d=False, moments=None):
    """G = 2(c 1^T + 1 c'^T) - 4 D_X T D_Y  (gw_grad_dp), in T's dtype (float32, or
    float64 = GW_F64 storage: k = 1 on 1-D supports).
    Sharded (ctx with a multi-rank comm): x, p are the full supports/marginals, T holds this
    rank's rows [row0, row0 + T.shape[0]) and the result holds the same rows of G.
    grid2d: x, y are the axes of 2-D grids with the Manhattan distance (GW_GRID2D).
    moments: optional (row_sum, row_ysum, col_sum, col_xsum) = (T 1, T y, T^T 1, T^T x) of the plan
    (gw_moments; this rank's rows / all rows), used for the totals instead of the reduced ones."""
    ctx = ctx or Context.get(T.device)
    dev = T.device
    x, y, p, q = (_vec(v, dev) for v in (x, y, p, q))
    ldT = _check_mat(T, "T")
    n, m = T.shape
    if out is None:
        out = plan_buffer(n, m, dev, T.dtype)
    ldG = _check_mat(out, "out", T.dtype)
    pr = _problem(x, y, p, q, n_local=n, row0=row0, flags=0 if validate else L.GW_NO_VALIDATE, k=k, grid2d=grid2d,
                  dtype=T.dtype)
    mom = None
    if moments is not None:
        mv = [_vec(v, dev) for v in moments]
        mom = L.gw_moments(*(v.data_ptr() for v in mv))
    L.check(ctx.lib.gw_grad_dp(ctx.h, C.byref(pr), _ptr(T), ldT, _ptr(out), ldG,
                               C.byref(mom) if mom is not None else None))
    return out


def sinkhorn(G, p, q, eps, max_iter, tol=0.0, check_every=10, f=None, g=None, return_plan=False, ctx=None):
    """Log-domain Sinkhorn on cost G (sinkhorn_solve).  Returns a dict with
    f, g (fp64 CUDA), iters, converged, violation and optionally T (G's dtype; float64 = GW_F64)."""
    ctx = ctx or Context.get(G.device)
    dev = G.device
    n, m = G.shape
    ldG = _check_mat(G, "G")
    p, q = _vec(p, dev), _vec(q, dev)
    # supports are irrelevant to Sinkhorn but the problem struct carries them: pass sorted dummies
    xs = torch.arange(n, dtype=torch.float64, device=dev)
    ys = torch.arange(m, dtype=torch.float64, device=dev)
    f = torch.zeros(n, dtype=torch.float64, device=dev) if f is None else _vec(f, dev).clone()
    g = torch.zeros(m, dtype=torch.float64, device=dev) if g is None else _vec(g, dev).clone()
    T = plan_buffer(n, m, dev, G.dtype) if return_plan else None
    pr = _problem(xs, ys, p, q, dtype=G.dtype)
    o = L.gw_sinkhorn_opts(eps, int(max_iter), float(tol), int(check_every))
    info = L.gw_sinkhorn_info()
    L.check(ctx.lib.sinkhorn_solve(ctx.h, C.byref(pr), _ptr(G), ldG, C.byref(o), _ptr(f), _ptr(g), _ptr(T),
                                   T.stride(0) if T is not None else 0, C.byref(info)))
    out = {"f": f, "g": g, "iters": info.iters, "converged": bool(info.converged),
           "violation": info.marginal_violation, "fused_iters": info.fused_iters}
    if return_plan:
        out["T"] = T
    return out


@dataclass
class Result:
    gw_objective: float
    entropic_objective: float
    marginal_violation: float
    outer_iters: int
    inner_iters_total: int
    converged: bool
    ms_grad: float
    ms_sinkhorn: float
    ms_total: float
    f: Optional[object] = None
    g: Optional[object] = None
    T: Optional[object] = None
    trace: Optional[np.ndarray] = None   # [outer, 4]: E(T^l), violation, inner iters, ms
    inner_fused_total: int = 0
    grad_onepass_total: int = 0          # gradients on the one-read (8 N M) path
    extra: dict = field(default_factory=dict)


def _result(res, f, g, T, tr):
    return Result(res.gw_objective, res.entropic_objective, res.marginal_violation, res.outer_iters,
                  res.inner_iters_total, bool(res.converged), res.ms_grad, res.ms_sinkhorn, res.ms_total,
                  f, g, T, tr, res.inner_fused_total, res.grad_onepass_total)


def _opts(eps, outer, inner, tol, check_every, trace_objective, tau=None):
    o = L.gw_solve_opts()
    o.eps = eps
    o.tau = eps if tau is None else float(tau)
    o.outer_iters = int(outer)
    o.inner = L.gw_sinkhorn_opts(eps, int(inner), float(tol), int(check_every))
    o.flags = L.GW_SOLVE_TRACE_OBJECTIVE if trace_objective else 0
    return o


def solve(x, y, p, q, eps, outer, inner, tol=0.0, check_every=10, T0=None, return_plan=False,
          trace_objective=False, fx=None, fy=None, alpha=None, device=None, ctx=None, row0=0, n_local=None, k=1,
          grid2d=False, tau=None, export_iter=0, export_T=None, export_G=None, dtype=torch.float32):
    """Entropic GW (entropic_gw_solve) or, with fx/fy/alpha, entropic FGW (fgw_solve), on
    device vectors; tau = eps.  Sharded (ctx with a multi-rank
    comm): x, p (and fx) are full; this rank owns rows [row0, row0 + n_local): f, T0 and the
    returned plan hold those rows, g is replicated, the objective and violation are global.
    grid2d: x, y are 2-D grid axes (GW_GRID2D); p, q have len(x)**2, len(y)**2 entries.
    tau: the mirror-descent step's KL weight (default eps, Remark 1): the
    subproblem is entropic OT of grad E + (eps - tau) ln T^l at regulariser tau (k = 1, 1-D).
    export_iter / export_T / export_G (debug, gw_solve_set_export): at outer iteration export_iter
    (1-based) write the plan T^{l-1} the gradient is evaluated on and the solver's own G^l into
    caller buffers (plan_buffer-shaped, same leading dimension).
    dtype: matrix storage, torch.float32 (default) or torch.float64 (GW_F64: T0, the returned plan and
    the export buffers are float64; k = 1 on 1-D supports; taken from T0 when given)."""
    dev = torch.device(device) if device is not None else (T0.device if T0 is not None else torch.device("cuda"))
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    ctx = ctx or Context.get(dev)
    x, y, p, q = (_vec(v, dev) for v in (x, y, p, q))
    n, m = p.numel(), q.numel()
    if n_local is not None:
        n = int(n_local)
    if T0 is not None:
        dtype = T0.dtype
    f = torch.empty(n, dtype=torch.float64, device=dev)
    g = torch.empty(m, dtype=torch.float64, device=dev)
    T = plan_buffer(n, m, dev, dtype) if return_plan else None
    ld = 0
    if T0 is not None:
        ld = _check_mat(T0, "T0")
        if T is not None and T.stride(0) != ld:
            T = torch.empty((n, ld), dtype=dtype, device=dev)[:, :m]
    elif T is not None:
        ld = T.stride(0)
    pr = _problem(x, y, p, q, n_local=n, row0=row0, k=k, grid2d=grid2d, dtype=dtype)
    o = _opts(eps, outer, inner, tol, check_every, trace_objective, tau)
    res = L.gw_result()
    tr = np.zeros((max(int(outer), 1), 4), dtype=np.float64)
    trp = tr.ctypes.data_as(C.c_void_p)
    if export_iter:
        bufs = [b for b in (export_T, export_G) if b is not None]
        eld = _check_mat(bufs[0], "export buffer", dtype) if bufs else 0
        for b in bufs:
            if b.stride(0) != eld:
                raise ValueError("export_T and export_G must share the leading dimension")
        L.check(ctx.lib.gw_solve_set_export(ctx.h, int(export_iter), _ptr(export_T), _ptr(export_G), eld))
    if fx is not None:
        fxv, fyv = _vec(fx, dev), _vec(fy, dev)
        L.check(ctx.lib.fgw_solve(ctx.h, C.byref(pr), _ptr(fxv), _ptr(fyv), float(alpha), C.byref(o), _ptr(T0),
                                  _ptr(T), ld, _ptr(f), _ptr(g), C.byref(res), trp))
    else:
        L.check(ctx.lib.entropic_gw_solve(ctx.h, C.byref(pr), C.byref(o), _ptr(T0), _ptr(T), ld, _ptr(f), _ptr(g),
                                          C.byref(res), trp))
    return _result(res, f, g, T, tr[: int(outer)])


def solve_host(x, y, p, q, eps, outer, inner, tol=0.0, check_every=10, device=None, ctx=None,
               fx=None, fy=None, alpha=None, row0=0, n_local=None, k=1, grid2d=False, tau=None, dtype=torch.float32):
    """entropic_gw_solve with HOST vectors (GW_HOST_VECTORS): the library stages x, y, p, q
    host->device and copies the duals f, g back.  This is the end-to-end public call.
    Sharded: as solve() (f holds this rank's n_local rows)."""
    ctx = ctx or Context.get(device)
    xs, ys, ps, qs = (np.ascontiguousarray(v, dtype=np.float64) for v in (x, y, p, q))
    n, m = ps.size, qs.size
    if grid2d and (n != xs.size ** 2 or m != ys.size ** 2):
        raise ValueError("grid2d: len(p) must be len(x)**2 and len(q) len(y)**2")
    nl = n if n_local is None else int(n_local)
    f = np.empty(nl)
    g = np.empty(m)
    pr = L.gw_problem()
    pr.n, pr.m, pr.row0, pr.n_local = n, m, int(row0), nl
    pr.x, pr.y, pr.p, pr.q = (a.ctypes.data for a in (xs, ys, ps, qs))
    pr.k, pr.loss, pr.dtype = int(k), L.GW_LOSS_SQUARE, _GW_DTYPE[dtype]
    pr.flags = L.GW_HOST_VECTORS | (L.GW_GRID2D if grid2d else 0)
    o = _opts(eps, outer, inner, tol, check_every, False, tau)
    res = L.gw_result()
    tr = np.zeros((max(int(outer), 1), 4))
    fp = f.ctypes.data_as(C.c_void_p)
    gp = g.ctypes.data_as(C.c_void_p)
    if fx is not None:
        fxs, fys = (np.ascontiguousarray(v, dtype=np.float64) for v in (fx, fy))
        L.check(ctx.lib.fgw_solve(ctx.h, C.byref(pr), fxs.ctypes.data_as(C.c_void_p),
                                  fys.ctypes.data_as(C.c_void_p), float(alpha), C.byref(o), None, None, 0, fp, gp,
                                  C.byref(res), tr.ctypes.data_as(C.c_void_p)))
    else:
        L.check(ctx.lib.entropic_gw_solve(ctx.h, C.byref(pr), C.byref(o), None, None, 0, fp, gp, C.byref(res),
                                          tr.ctypes.data_as(C.c_void_p)))
    return _result(res, f, g, None, tr[: int(outer)])


def ugw_solve(x, y, u, v, rho, eps, outer, inner, trace_objective=False, return_plan=False, device=None, ctx=None,
              k=1, row0=0, n_local=None):
    """Entropic unbalanced GW (ugw_solve; Remark 3, readings R32-R35 in DESIGN.md)
    on device vectors.  Returns a Result: gw_objective = E(T), entropic_objective = F_eps(T),
    trace [outer, 4] = {F_eps, E, inner iterations, mass}."""
    dev = torch.device(device) if device is not None else torch.device("cuda")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    ctx = ctx or Context.get(dev)
    x, y, u, v = (_vec(t, dev) for t in (x, y, u, v))
    n, m = u.numel(), v.numel()
    if n_local is not None:
        n = int(n_local)
    f = torch.empty(n, dtype=torch.float64, device=dev)
    g = torch.empty(m, dtype=torch.float64, device=dev)
    T = plan_buffer(n, m, dev) if return_plan else None
    pr = _problem(x, y, u, v, n_local=n, row0=row0, k=k)
    o = _opts(eps, outer, inner, 0.0, 10, trace_objective)
    res = L.gw_result()
    tr = np.zeros((max(int(outer), 1), 4), dtype=np.float64)
    L.check(ctx.lib.ugw_solve(ctx.h, C.byref(pr), float(rho), C.byref(o), None, _ptr(T),
                              T.stride(0) if T is not None else 0, _ptr(f), _ptr(g), C.byref(res),
                              tr.ctypes.data_as(C.c_void_p)))
    return _result(res, f, g, T, tr[: int(outer)])
