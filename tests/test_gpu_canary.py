"""Out-of-bounds write and input-mutation check by canaries (compute-sanitizer is closed on this GPU pool, so
this stands in for memcheck on the matrices the caller owns): every N x M matrix handed to the C ABI lives
inside a larger allocation -- 8 guard rows above and below, padding columns [m, ld) -- pre-filled with a
sentinel bit pattern.  After each call: the guard rows of every matrix and the padding of every INPUT matrix
are bitwise intact, inputs are bitwise unchanged ("Inputs are never mutated", include/gwdp.h), and outputs are
finite on [0, n) x [0, m).  Shapes are ragged (m % 4 != 0, rows not a multiple of any tile height)."""

import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu

GUARD = 8
SENT32 = 0x7FC12345          # a quiet NaN with a payload
SENT64 = 0x7FF8123456789ABC


@pytest.fixture(scope="module")
def gw():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as ge
    ge.build()
    from paper_2404_08970_b200 import api
    return api


class Guarded:
    """An (n, m) matrix view inside a sentinel-filled (n + 2 GUARD, ld) allocation."""

    def __init__(self, n, m, dtype, dev):
        import torch
        self.n, self.m = n, m
        self.ld = (m + 31) // 32 * 32 + 32            # at least 32 padding columns
        it, sent = (torch.int32, SENT32) if dtype == torch.float32 else (torch.int64, SENT64)
        self.sent = sent
        self.raw = torch.full((n + 2 * GUARD, self.ld), sent, dtype=it, device=dev)
        self.all = self.raw.view(dtype)
        self.view = self.all[GUARD:GUARD + n, :m]

    def guards_intact(self):
        r = self.raw
        return bool((r[:GUARD] == self.sent).all() and (r[GUARD + self.n:] == self.sent).all())

    def padding_intact(self):
        return bool((self.raw[GUARD:GUARD + self.n, self.m:] == self.sent).all())

    def snapshot(self):
        return self.raw.clone()

    def unchanged(self, snap):
        return bool((self.raw == snap).all())


def _plan(rng, n, m):
    T = rng.random((n, m)) + 0.05
    return T / T.sum()


@pytest.mark.parametrize("n,m", [(1, 1), (37, 53), (300, 517), (1000, 777), (130, 9001), (64, 1003), (50, 1002),
                                 (513, 4099)])
@pytest.mark.parametrize("k", [1, 2, 3])
def test_grad_fp32_canaries(gw, n, m, k):
    import torch
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(n * 1000 + m + k)
    x, y = np.sort(rng.random(n)), np.sort(rng.random(m))
    p, q = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
    T, G = Guarded(n, m, torch.float32, dev), Guarded(n, m, torch.float32, dev)
    T.view.copy_(torch.from_numpy(_plan(rng, n, m)))
    snap = T.snapshot()
    gw.grad(x, y, p, q, T.view, out=G.view, k=k)
    torch.cuda.synchronize()
    assert T.unchanged(snap), "gw_grad_dp mutated its input plan (or its guards / padding)"
    assert G.guards_intact(), "gw_grad_dp wrote outside the rows of G"
    assert G.padding_intact(), "gw_grad_dp wrote into the padding columns [m, ld) of G"
    assert bool(torch.isfinite(G.view).all())


@pytest.mark.parametrize("n,m,k", [(1, 1, 1), (133, 70, 1), (300, 257, 1), (257, 300, 3), (64, 1000, 2),
                                   (90, 1003, 1), (90, 1003, 2)])
def test_grad_fp64_canaries(gw, n, m, k):
    import torch
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(n * 1000 + m + k)
    x, y = np.sort(rng.random(n)), np.sort(rng.random(m))
    p, q = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
    T, G = Guarded(n, m, torch.float64, dev), Guarded(n, m, torch.float64, dev)
    T.view.copy_(torch.from_numpy(_plan(rng, n, m)))
    snap = T.snapshot()
    gw.grad(x, y, p, q, T.view, out=G.view, k=k)
    torch.cuda.synchronize()
    assert T.unchanged(snap)
    assert G.guards_intact() and G.padding_intact()
    assert bool(torch.isfinite(G.view).all())


@pytest.mark.parametrize("sx,sy", [(1, 1), (5, 7), (12, 9), (6, 33)])
def test_grad_grid2d_canaries(gw, sx, sy):
    import torch
    dev = torch.device("cuda", 0)
    n, m = sx * sx, sy * sy
    rng = np.random.default_rng(sx * 100 + sy)
    ax, ay = np.arange(sx) / max(sx - 1, 1), np.arange(sy) / max(sy - 1, 1)
    p, q = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
    T, G = Guarded(n, m, torch.float32, dev), Guarded(n, m, torch.float32, dev)
    T.view.copy_(torch.from_numpy(_plan(rng, n, m)))
    snap = T.snapshot()
    gw.grad(ax, ay, p, q, T.view, out=G.view, grid2d=True)
    torch.cuda.synchronize()
    assert T.unchanged(snap)
    assert G.guards_intact() and G.padding_intact()
    assert bool(torch.isfinite(G.view).all())


@pytest.mark.parametrize("n,m", [(5, 3), (200, 150), (40, 9001), (700, 1030)])
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_sinkhorn_and_solve_canaries(gw, n, m, dtype):
    import torch
    dev = torch.device("cuda", 0)
    dt = torch.float32 if dtype == "f32" else torch.float64
    P = W.config5(n, m)
    rng = np.random.default_rng(n + m)
    # sinkhorn_solve: the cost is an input
    Gc = Guarded(n, m, dt, dev)
    Gc.view.copy_(torch.from_numpy(rng.random((n, m))))
    snap = Gc.snapshot()
    r = gw.sinkhorn(Gc.view, P.p, P.q, 0.05, 12, return_plan=True)
    torch.cuda.synchronize()
    assert Gc.unchanged(snap), "sinkhorn_solve mutated its cost (or its guards / padding)"
    assert bool(torch.isfinite(r["T"]).all())
    # entropic_gw_solve: T0 is an input, the export buffers are outputs
    T0 = Guarded(n, m, dt, dev)
    T0.view.copy_(torch.from_numpy(np.outer(P.p, P.q)))
    snap0 = T0.snapshot()
    eT, eG = Guarded(n, m, dt, dev), Guarded(n, m, dt, dev)
    assert eT.ld == eG.ld
    r = gw.solve(P.x, P.y, P.p, P.q, 0.02, 2, 15, T0=T0.view, return_plan=True, device=dev, dtype=dt,
                 export_iter=2, export_T=eT.view, export_G=eG.view)
    torch.cuda.synchronize()
    assert T0.unchanged(snap0), "entropic_gw_solve mutated T0 (or its guards / padding)"
    assert eT.guards_intact() and eG.guards_intact()
    assert eT.padding_intact() and eG.padding_intact()  # the export is a 2-D copy of [0, n) x [0, m)
    assert bool(torch.isfinite(eT.view).all()) and bool(torch.isfinite(eG.view).all())
    assert bool(torch.isfinite(r.T).all())
    if dtype == "f32":  # FGW through the same entry point (feature term fused into the gradient kernels)
        eG2 = Guarded(n, m, dt, dev)
        gw.solve(P.x, P.y, P.p, P.q, 0.02, 2, 15, fx=P.fx, fy=P.fy, alpha=0.5, device=dev, export_iter=2,
                 export_G=eG2.view)
        torch.cuda.synchronize()
        assert eG2.guards_intact() and eG2.padding_intact()
        assert bool(torch.isfinite(eG2.view).all())


def test_validation_errors_write_nothing(gw):
    """include/gwdp.h: "Argument and validation errors are detected before any output is written"."""
    import torch
    from paper_2404_08970_b200 import GwError
    dev = torch.device("cuda", 0)
    n, m = 120, 77
    rng = np.random.default_rng(5)
    x, y = np.sort(rng.random(n)), np.sort(rng.random(m))
    p, q = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
    T, G = Guarded(n, m, torch.float32, dev), Guarded(n, m, torch.float32, dev)
    T.view.copy_(torch.from_numpy(_plan(rng, n, m)))
    g0 = G.snapshot()
    bad_x = x.copy()
    bad_x[[3, 4]] = bad_x[[4, 3]]                      # unsorted support
    bad_p = p.copy()
    bad_p[7] = -bad_p[7]                               # negative mass
    for args in ((bad_x, y, p, q), (x, y, bad_p, q), (x, y, 2.0 * p, q)):
        with pytest.raises(GwError):
            gw.grad(*args, T.view, out=G.view)
        torch.cuda.synchronize()
        assert G.unchanged(g0), "gw_grad_dp wrote into G before rejecting its arguments"
    eT, eG = Guarded(n, m, torch.float32, dev), Guarded(n, m, torch.float32, dev)
    t0, g1 = eT.snapshot(), eG.snapshot()
    with pytest.raises(GwError):
        gw.solve(bad_x, y, p, q, 0.02, 2, 10, device=dev, export_iter=1, export_T=eT.view, export_G=eG.view)
    torch.cuda.synchronize()
    assert eT.unchanged(t0) and eG.unchanged(g1)
    # the rejected call consumed its one-shot export request: the next valid solve exports nothing
    gw.solve(x, y, p, q, 0.02, 2, 10, device=dev)
    torch.cuda.synchronize()
    assert eT.unchanged(t0) and eG.unchanged(g1)
