"""GW_F64 storage (f64.cuh): every N x M matrix float64 and every step in fp64 (C1 = BASELINE
configs[0], whose matrices SURVEY.md §8's sizes table puts in fp64).  Parity against the float64
oracle is then at rounding level, not at the north_star's fp32-storage tolerances:
  gradient max-abs error <= GRAD64_TOL * max|G| (the DP's fp64 prefix sums vs two dense DGEMMs),
  Sinkhorn duals / eps and plan / max T <= SINK64_TOL (fp64 LSEs in a different summation order),
  solver objective trajectory (C1: 20 x 100) relative <= OBJ64_TOL.
The tolerances are about 10x the largest errors measured on a B200 (GW_F64)."""

import json
import os

import numpy as np
import pytest

import oracle as O
import workloads as W

pytestmark = pytest.mark.gpu

GRAD64_TOL = 1e-13
SINK64_TOL = 5e-13
OBJ64_TOL = 3e-12
VIOL64_TOL = 1e-12

_LOG = os.environ.get("GWDP_F64_LOG")


def _log(**kw):
    if _LOG:
        with open(_LOG, "a") as fh:
            fh.write(json.dumps(kw) + "\n")


@pytest.fixture(scope="module")
def gw():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as ge
    ge.build()
    from paper_2404_08970_b200 import api
    return api


def _dev():
    import torch
    return torch.device("cuda", 0)


def _to_dev64(api, A):
    import torch
    n, m = A.shape
    t = api.plan_buffer(n, m, _dev(), torch.float64)
    t.copy_(torch.from_numpy(np.ascontiguousarray(A, dtype=np.float64)))
    return t


def _np(t):
    return t.cpu().numpy().astype(np.float64)


def _rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


SHAPES = [(1, 1), (1, 7), (7, 1), (3, 5), (64, 64), (65, 129), (255, 300), (256, 256), (600, 1000), (1000, 777)]


@pytest.mark.parametrize("n,m", SHAPES)
def test_grad64_random_plan(gw, n, m):
    """gw_grad_dp (GW_F64) vs grad_prescribed (two dense DGEMMs): ragged row blocks
    (64 rows) and warp chunks (32 columns), padded ld."""
    rng = np.random.default_rng(1000 * n + m)
    x, y = np.sort(rng.random(n)), np.sort(rng.random(m))
    p, q = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
    Tn = rng.exponential(size=(n, m)) / (n * m)
    G = _np(gw.grad(x, y, p, q, _to_dev64(gw, Tn)))
    Go = O.grad_prescribed(x, y, p, q, Tn)
    err = _rel(G, Go)
    _log(test="grad64", n=n, m=m, err=err)
    assert err <= GRAD64_TOL


def test_grad64_ties_and_translation(gw):
    """Tied supports (x_i = x_j: zero gaps in the scans) and a large common offset (centring)."""
    rng = np.random.default_rng(5)
    n, m = 300, 200
    x = np.sort(np.round(rng.random(n) * 20) / 20) + 1e3
    y = np.sort(np.round(rng.random(m) * 10) / 10) - 7.0
    p, q = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
    Tn = rng.random((n, m)) / (n * m)
    G = _np(gw.grad(x, y, p, q, _to_dev64(gw, Tn)))
    Go = O.grad_prescribed(x, y, p, q, Tn)
    err = _rel(G, Go)
    _log(test="grad64_ties", err=err)
    assert err <= GRAD64_TOL


def test_grad64_in_place_and_moments(gw):
    """G aliasing T (ldG == ldT) and supplied gw_moments give the same G (up to the totals' rounding)."""
    rng = np.random.default_rng(11)
    n, m = 333, 257
    x, y = np.sort(rng.random(n)), np.sort(rng.random(m))
    p, q = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
    Tn = rng.random((n, m)) / (n * m)
    Go = O.grad_prescribed(x, y, p, q, Tn)
    T = _to_dev64(gw, Tn)
    ref = _np(gw.grad(x, y, p, q, T))
    mom = (Tn.sum(1), Tn @ y, Tn.sum(0), Tn.T @ x)
    Gm = _np(gw.grad(x, y, p, q, T, moments=mom))
    gw.grad(x, y, p, q, T, out=T)
    Gi = _np(T)
    np.testing.assert_array_equal(Gi, ref)
    assert _rel(Gm, Go) <= GRAD64_TOL
    assert _rel(ref, Go) <= GRAD64_TOL


def test_grad64_product_closed_form(gw):
    """On T = p q^T the gradient is 2c_i + 2c'_p - 4 (D_X p)_i (D_Y q)_p (closed form P7)."""
    rng = np.random.default_rng(3)
    n, m = 200, 150
    x, y = np.sort(rng.random(n)), np.sort(rng.random(m))
    p, q = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
    G = _np(gw.grad(x, y, p, q, _to_dev64(gw, np.outer(p, q))))
    DX, DY = np.abs(x[:, None] - x[None, :]), np.abs(y[:, None] - y[None, :])
    c, c2 = (DX * DX) @ p, (DY * DY) @ q
    Gc = 2 * c[:, None] + 2 * c2[None, :] - 4 * np.outer(DX @ p, DY @ q)
    assert _rel(G, Gc) <= GRAD64_TOL


@pytest.mark.parametrize("n,m", [(1, 1), (5, 3), (64, 65), (256, 256), (300, 700)])
def test_sinkhorn64(gw, n, m):
    """sinkhorn_solve (GW_F64) vs the oracle's log-domain Sinkhorn: duals, plan,
    violation, warm start."""
    rng = np.random.default_rng(7 * n + m)
    x, y = np.sort(rng.random(n)), np.sort(rng.random(m))
    p, q = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
    G = O.grad_prescribed(x, y, p, q, np.outer(p, q))
    eps = 0.02
    f0, g0 = rng.normal(size=n) * eps, rng.normal(size=m) * eps
    r = gw.sinkhorn(_to_dev64(gw, G), p, q, eps, 60, f=f0, g=g0, return_plan=True)
    fo, go, _ = O.sinkhorn(G, p, q, eps, 60, f0=f0, g0=g0)
    Tn = O.plan_from_duals(G, fo, go, eps)
    ef = float(np.max(np.abs(_np(r["f"]) - fo)) / eps)
    eg = float(np.max(np.abs(_np(r["g"]) - go)) / eps)
    eT = _rel(_np(r["T"]), Tn)
    _log(test="sinkhorn64", n=n, m=m, ef=ef, eg=eg, eT=eT)
    assert max(ef, eg, eT) <= SINK64_TOL
    assert abs(r["violation"] - O.violation(Tn, p, q)) <= VIOL64_TOL
    assert r["fused_iters"] == 0


def test_sinkhorn64_tolerance_rule(gw):
    """tol > 0: the violation checked every check_every iterations, same stopping count as the oracle."""
    P = W.config1()
    G = O.grad_prescribed(P.x, P.y, P.p, P.q, np.outer(P.p, P.q))
    tol = 1e-9
    r = gw.sinkhorn(_to_dev64(gw, G), P.p, P.q, P.eps, 2000, tol=tol, check_every=10)
    fo, go, used = O.sinkhorn(G, P.p, P.q, P.eps, 2000, tol=tol, check_every=10)
    _log(test="sinkhorn64_tol", iters=r["iters"], used=used, ef=float(np.max(np.abs(_np(r["f"]) - fo)) / P.eps))
    assert r["iters"] == used
    assert r["converged"] and r["violation"] <= tol
    assert np.max(np.abs(_np(r["f"]) - fo)) / P.eps <= SINK64_TOL


def test_solver64_c1_trajectory(gw):
    """C1 (BASELINE configs[0]) with its fp64 matrices: N = M = 256, eps = 1e-2, 20 outer x 100 inner,
    T0 = p q^T.  Every outer iteration's E(T^l), the final objective, entropic objective, plan,
    duals and violation against the oracle at rounding level."""
    import torch
    P = W.config1()
    r = gw.solve(P.x, P.y, P.p, P.q, P.eps, P.outer, P.inner, trace_objective=True, return_plan=True,
                 dtype=torch.float64)
    ro = O.entropic_gw(P.x, P.y, P.p, P.q, P.eps, P.outer, P.inner)
    eE = float(np.max(np.abs(r.trace[:, 0] - ro["E"]) / np.abs(ro["E"])))
    eobj = abs(r.gw_objective - ro["gw_objective"]) / abs(ro["gw_objective"])
    eent = abs(r.entropic_objective - ro["entropic_objective"]) / abs(ro["entropic_objective"])
    T = _np(r.T)
    eT = _rel(T, ro["T"])
    ef = float(np.max(np.abs(_np(r.f) - ro["f"])) / P.eps)
    ev = abs(r.marginal_violation - ro["viol"][-1])
    _log(test="solver64_c1", eE=eE, eobj=eobj, eent=eent, eT=eT, ef=ef, ev=ev, viol=r.marginal_violation)
    assert r.T.dtype == torch.float64
    assert max(eE, eobj, eent) <= OBJ64_TOL
    assert max(eT, ef) <= OBJ64_TOL
    assert ev <= VIOL64_TOL
    assert np.max(np.abs(r.trace[:, 1] - ro["viol"])) <= VIOL64_TOL
    assert abs(O.objective(P.x, P.y, T) - r.gw_objective) <= OBJ64_TOL * abs(r.gw_objective)


def test_solver64_fgw(gw):
    """Entropic FGW (Remark 2) with fp64 storage vs entropic_fgw."""
    import torch
    rng = np.random.default_rng(21)
    n, m = 200, 150
    x, y = np.sort(rng.beta(2, 5, n)), np.sort(rng.beta(5, 2, m))
    p, q = rng.dirichlet(np.full(n, 0.5)), rng.dirichlet(np.full(m, 0.5))
    fx, fy = rng.normal(size=n), rng.normal(size=m)
    eps = 0.05
    r = gw.solve(x, y, p, q, eps, 4, 50, fx=fx, fy=fy, alpha=0.5, trace_objective=True, dtype=torch.float64)
    ro = O.entropic_fgw(x, y, p, q, fx, fy, 0.5, eps, 4, 50)
    eE = float(np.max(np.abs(r.trace[:, 0] - ro["E"]) / np.abs(ro["E"])))
    _log(test="solver64_fgw", eE=eE)
    assert eE <= OBJ64_TOL
    assert abs(r.entropic_objective - ro["entropic_objective"]) <= OBJ64_TOL * abs(ro["entropic_objective"])


def test_solver64_tol_and_T0(gw):
    """Inner tolerance rule (reading R8) and an explicit T0; outer = 0 returns T0 and its objective."""
    import torch
    rng = np.random.default_rng(4)
    n, m = 128, 96
    x, y = np.sort(rng.random(n)), np.sort(rng.random(m))
    p, q = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
    T0n = rng.random((n, m))
    T0n = T0n / T0n.sum()
    T0 = _to_dev64(gw, T0n)
    r = gw.solve(x, y, p, q, 0.02, 3, 500, tol=1e-10, check_every=10, T0=T0, trace_objective=True)
    ro = O.entropic_gw(x, y, p, q, 0.02, 3, 500, T0=T0n, tol=1e-10, check_every=10)
    np.testing.assert_array_equal(r.trace[:, 2], ro["inner_used"])
    assert np.max(np.abs(r.trace[:, 0] - ro["E"]) / np.abs(ro["E"])) <= OBJ64_TOL
    r0 = gw.solve(x, y, p, q, 0.02, 0, 10, T0=T0, return_plan=True)
    np.testing.assert_array_equal(_np(r0.T), T0n)
    assert abs(r0.gw_objective - O.objective(x, y, T0n)) <= OBJ64_TOL * abs(r0.gw_objective)


def test_solver64_export_and_host(gw):
    """The debug export writes fp64 T^{l-1} and G^l; the host-vector entry point agrees with the device one."""
    import torch
    P = W.config1()
    n, m = P.x.size, P.y.size
    Te = gw.plan_buffer(n, m, _dev(), torch.float64)
    Ge = gw.plan_buffer(n, m, _dev(), torch.float64)
    r = gw.solve(P.x, P.y, P.p, P.q, P.eps, 3, 100, dtype=torch.float64, export_iter=2, export_T=Te, export_G=Ge)
    Tn = _np(Te)
    assert _rel(_np(Ge), O.grad_prescribed(P.x, P.y, P.p, P.q, Tn)) <= GRAD64_TOL
    ro = O.entropic_gw(P.x, P.y, P.p, P.q, P.eps, 1, 100)
    assert _rel(Tn, ro["T"]) <= OBJ64_TOL
    rh = gw.solve_host(P.x, P.y, P.p, P.q, P.eps, 3, 100, dtype=torch.float64)
    assert abs(rh.gw_objective - r.gw_objective) <= 1e-14 * abs(r.gw_objective)
    np.testing.assert_allclose(rh.g, _np(r.g), rtol=0, atol=1e-14)


def test_f64_unsupported(gw):
    """GW_F64 is 1-D supports (k = 1..5): 2-D grids and tau != eps are rejected."""
    import torch
    from paper_2404_08970_b200 import _lib as L
    rng = np.random.default_rng(0)
    x, y = np.sort(rng.random(16)), np.sort(rng.random(16))
    p = q = np.full(16, 1 / 16)
    T = _to_dev64(gw, np.outer(p, q))
    with pytest.raises(L.GwError) as e:
        gw.grad(np.arange(4.0), np.arange(4.0), p, q, T, grid2d=True)
    assert e.value.code == "GW_ERR_UNSUPPORTED"
    with pytest.raises(L.GwError) as e:
        gw.solve(x, y, p, q, 0.1, 1, 5, tau=0.05, dtype=torch.float64)
    assert e.value.code == "GW_ERR_UNSUPPORTED"
    with pytest.raises(ValueError):  # mixed storage in one call
        gw.grad(x, y, p, q, T, out=gw.plan_buffer(16, 16, _dev()))


@pytest.mark.parametrize("R", [2, 3])
def test_sharded64(gw, R, monkeypatch):
    """Row-sharded GW_F64 (R threads on one GPU, host-callback all-gathers): the
    gradient rows and the solve's objective, duals and violation equal the single-rank ones up to
    summation order and the oracle at rounding level."""
    import torch
    from paper_2404_08970_b200 import dist
    from test_gpu_sharded import _run_ranks
    monkeypatch.setenv("GWDP_NO_SMALL", "1")
    rng = np.random.default_rng(70 + R)
    n, m = 333, 190  # several 64-row blocks per rank, ragged
    x, y = np.sort(rng.random(n)), np.sort(rng.random(m))
    p, q = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
    Tn = rng.exponential(size=(n, m)) / (n * m)
    T = _to_dev64(gw, Tn)
    Go = O.grad_prescribed(x, y, p, q, Tn)

    def fg(r, ctx, st):
        r0, nl = dist.shard_rows(n, R, r)
        return r0, _np(gw.grad(x, y, p, q, T[r0:r0 + nl], ctx=ctx, row0=r0))

    Gs = np.concatenate([g for _, g in sorted(_run_ranks(R, fg), key=lambda t: t[0])])
    assert _rel(Gs, Go) <= GRAD64_TOL
    P = W.config5(240, 200)
    eps = P.eps
    r1 = gw.solve(P.x, P.y, P.p, P.q, eps, 4, 60, dtype=torch.float64)
    ro = O.entropic_gw(P.x, P.y, P.p, P.q, eps, 4, 60)

    def fs(r, ctx, st):
        r0, nl = dist.shard_rows(P.x.size, R, r)
        res = gw.solve(P.x, P.y, P.p, P.q, eps, 4, 60, ctx=ctx, row0=r0, n_local=nl, device=ctx.device,
                       dtype=torch.float64)
        return r0, res.gw_objective, res.marginal_violation, _np(res.f), _np(res.g)

    out = _run_ranks(R, fs)
    assert len({o[1] for o in out}) == 1, "every rank reports the same global objective"
    assert abs(out[0][1] - r1.gw_objective) <= 1e-12 * abs(r1.gw_objective)
    assert abs(out[0][1] - ro["gw_objective"]) <= OBJ64_TOL * abs(ro["gw_objective"])
    for o in out[1:]:
        np.testing.assert_array_equal(o[4], out[0][4])
    f = np.concatenate([o[3] for o in sorted(out, key=lambda t: t[0])])
    ef = float(np.max(np.abs(f - _np(r1.f))) / eps)
    eo = abs(out[0][1] - ro["gw_objective"]) / abs(ro["gw_objective"])
    _log(test="sharded64", R=R, ef=ef, eo=eo, eg=_rel(Gs, Go))
    assert ef <= SINK64_TOL


def test_solver64_degenerate(gw):
    """Degenerate inputs on the fp64 path: zero-mass rows and columns (ln 0 = -inf duals, empty plan rows),
    a single point on either side (n = 1 or m = 1: the plan is p q^T), against the oracle."""
    import torch
    rng = np.random.default_rng(9)
    n, m = 70, 45
    x, y = np.sort(rng.random(n)), np.sort(rng.random(m))
    p, q = rng.random(n), rng.random(m)
    p[[0, 13, 69]] = 0.0
    q[[5, 44]] = 0.0
    p, q = p / p.sum(), q / q.sum()
    r = gw.solve(x, y, p, q, 0.05, 3, 40, trace_objective=True, return_plan=True, dtype=torch.float64)
    ro = O.entropic_gw(x, y, p, q, 0.05, 3, 40)
    T = _np(r.T)
    assert np.all(T[[0, 13, 69], :] == 0.0) and np.all(T[:, [5, 44]] == 0.0)
    assert _rel(T, ro["T"]) <= OBJ64_TOL
    assert np.max(np.abs(r.trace[:, 0] - ro["E"]) / np.abs(ro["E"])) <= OBJ64_TOL
    assert abs(r.entropic_objective - ro["entropic_objective"]) <= OBJ64_TOL * abs(ro["entropic_objective"])
    for (a, b) in [(1, 9), (9, 1)]:
        xa, yb = np.sort(rng.random(a)), np.sort(rng.random(b))
        pa, qb = rng.dirichlet(np.ones(a)), rng.dirichlet(np.ones(b))
        r1 = gw.solve(xa, yb, pa, qb, 0.05, 2, 10, return_plan=True, dtype=torch.float64)
        assert _rel(_np(r1.T), np.outer(pa, qb)) <= 1e-14
        assert abs(r1.gw_objective - O.objective(xa, yb, np.outer(pa, qb))) <= 1e-14 + 1e-12 * abs(r1.gw_objective)


@pytest.mark.parametrize("k", [2, 3, 4, 5])
@pytest.mark.parametrize("n,m", [(1, 1), (7, 3), (65, 129), (300, 257)])
def test_grad64_power_k(gw, k, n, m):
    """Distance powers k = 2..5 (reading R17) with fp64 storage: the k + 1 power-sum
    scans (odd k) or totals (even k) vs grad_prescribed(k) (two dense DGEMMs)."""
    rng = np.random.default_rng(100 * k + n + m)
    x, y = np.sort(rng.random(n)), np.sort(rng.random(m))
    p, q = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
    Tn = rng.exponential(size=(n, m)) / (n * m)
    G = _np(gw.grad(x, y, p, q, _to_dev64(gw, Tn), k=k))
    Go = O.grad_prescribed(x, y, p, q, Tn, k)
    err = _rel(G, Go)
    _log(test="grad64_k", k=k, n=n, m=m, err=err)
    assert err <= GRAD64_TOL


@pytest.mark.parametrize("k", [2, 3, 5])
def test_solver64_power_k(gw, k):
    """Entropic GW with |x - x'|^k (k = 2, 3, 5) and fp64 storage: trajectory against the oracle."""
    import torch
    P = W.config5(150, 120)
    r = gw.solve(P.x, P.y, P.p, P.q, 0.02, 4, 60, k=k, trace_objective=True, dtype=torch.float64)
    ro = O.entropic_gw(P.x, P.y, P.p, P.q, 0.02, 4, 60, k=k)
    eE = float(np.max(np.abs(r.trace[:, 0] - ro["E"]) / np.abs(ro["E"])))
    _log(test="solver64_k", k=k, eE=eE)
    assert eE <= OBJ64_TOL
    assert abs(r.entropic_objective - ro["entropic_objective"]) <= OBJ64_TOL * abs(ro["entropic_objective"])


@pytest.mark.parametrize("n,m", [(256, 256), (37, 300), (300, 5)])
def test_solver64_small_vs_multikernel(gw, n, m, monkeypatch):
    """The cluster-resident fp64 Sinkhorn (k64_sink_small: every inner iteration in one launch) and the
    multi-kernel route (GWDP_NO_SMALL=1: row LSE, column partials, merge; graph-replayed) against each
    other and the oracle."""
    import torch
    rng = np.random.default_rng(n + 7 * m)
    x, y = np.sort(rng.random(n)), np.sort(rng.random(m))
    p, q = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
    r_small = gw.solve(x, y, p, q, 0.01, 5, 100, trace_objective=True, dtype=torch.float64)
    monkeypatch.setenv("GWDP_NO_SMALL", "1")
    r_multi = gw.solve(x, y, p, q, 0.01, 5, 100, trace_objective=True, dtype=torch.float64)
    ro = O.entropic_gw(x, y, p, q, 0.01, 5, 100)
    es = float(np.max(np.abs(r_small.trace[:, 0] - ro["E"]) / np.abs(ro["E"])))
    em = float(np.max(np.abs(r_multi.trace[:, 0] - ro["E"]) / np.abs(ro["E"])))
    ef = float(np.max(np.abs(_np(r_small.f) - _np(r_multi.f))) / 0.01)
    _log(test="small_vs_multi64", n=n, m=m, es=es, em=em, ef=ef)
    assert max(es, em) <= OBJ64_TOL
    assert ef <= OBJ64_TOL
