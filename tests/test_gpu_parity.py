"""GPU parity: the CUDA path (through the C ABI) against the float64 oracle on the same
seeded inputs.  Tolerances are the north_star's (BASELINE.json):
  gradient max-abs error <= 1e-5 * max|G|,  final GW objective rel. error <= 1e-4,
  marginal violation <= 1e-6.
"""

import numpy as np
import pytest

import oracle as O
import workloads as W

pytestmark = pytest.mark.gpu

GRAD_TOL = 1e-5
OBJ_TOL = 1e-4
VIOL_TOL = 1e-6
# Sinkhorn (60 iterations on an fp32 cost, fp32 exponents): plan error / max T and dual error / eps,
# ~3x the largest values measured on a B200 (round 2: plan 1.0e-6 at 64 x 65536, duals 9.7e-7)
PLAN_TOL = 3e-6
DUAL_TOL = 3e-6


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


def _to_dev(api, T):
    import torch
    n, m = T.shape
    t = api.plan_buffer(n, m, _dev())
    t.copy_(torch.from_numpy(np.ascontiguousarray(T, dtype=np.float32)))
    return t


def _grad_err(G, Go):
    return np.max(np.abs(G - Go)) / max(np.max(np.abs(Go)), 1e-300)


# ----------------------------------------------------------------------------- gradient

GRAD_SHAPES = [(1, 1), (1, 7), (7, 1), (3, 5), (64, 64), (255, 300), (256, 256), (257, 513), (600, 1000),
               (1000, 777), (1024, 1031)]


@pytest.mark.parametrize("n,m", GRAD_SHAPES)
def test_grad_random_plan(gw, n, m):
    """gw_grad_dp vs grad_prescribed on a random fp32 plan, ragged tails,
    ties in the supports, non-uniform marginals."""
    rng = np.random.default_rng(n * 1000 + m)
    x, y = np.sort(rng.random(n)), np.sort(rng.random(m))
    if n > 10:
        x[5] = x[4]
    if m > 10:
        y[7] = y[6]
    p, q = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
    T = (rng.exponential(size=(n, m)) / (n * m)).astype(np.float32)
    G = gw.grad(x, y, p, q, _to_dev(gw, T)).cpu().numpy().astype(np.float64)
    Go = O.grad_prescribed(x, y, p, q, T.astype(np.float64))
    assert _grad_err(G, Go) <= GRAD_TOL


def test_grad_c3_recipe_4096(gw):
    """C3 recipe (Exp(1) rescaled to uniform marginals) at N = M = 4096, full matrix."""
    P = W.config3(4096)
    T = P.extra["T"]
    G = gw.grad(P.x, P.y, P.p, P.q, _to_dev(gw, T)).cpu().numpy().astype(np.float64)
    Go = O.grad_prescribed(P.x, P.y, P.p, P.q, T.astype(np.float64))
    assert _grad_err(G, Go) <= GRAD_TOL


def test_grad_product_closed_form(gw):
    """At T0 = p (x) q the gradient is G0 = 2(c_i + c'_p) - 4 (D_X p)_i (D_Y q)_p (P7)."""
    P = W.uniform_problem(777, 1290, seed=3)
    T = np.outer(P.p, P.q).astype(np.float32)
    G = gw.grad(P.x, P.y, P.p, P.q, _to_dev(gw, T)).cpu().numpy().astype(np.float64)
    DX, DY = O.dist(P.x), O.dist(P.y)
    Tq = T.astype(np.float64)
    a, b = Tq.sum(1), Tq.sum(0)
    c, c2 = O.const_term(P.x, P.y, P.p, P.q)
    G0 = 2 * (c[:, None] + c2[None, :]) - 4 * np.outer(DX @ a, DY @ b)
    assert _grad_err(G, G0) <= GRAD_TOL


def test_grad_in_place(gw):
    rng = np.random.default_rng(5)
    n, m = 300, 400
    x, y = np.sort(rng.random(n)), np.sort(rng.random(m))
    p, q = np.full(n, 1 / n), np.full(m, 1 / m)
    T = (rng.random((n, m)) / (n * m)).astype(np.float32)
    Td = _to_dev(gw, T)
    G = gw.grad(x, y, p, q, Td, out=Td).cpu().numpy().astype(np.float64)
    assert _grad_err(G, O.grad_prescribed(x, y, p, q, T.astype(np.float64))) <= GRAD_TOL


def test_grad_supplied_moments(gw):
    """gw_grad_dp with gw_moments (the plan's T1, Ty, T^T 1, T^T x in the caller's coordinates): the
    totals are taken from the argument -- exact moments give the same G (both at the tolerance of the
    dense definition), perturbed ones move G (so they are used), null members are rejected."""
    import torch
    from paper_2404_08970_b200 import GwError
    rng = np.random.default_rng(77)
    n, m = 600, 700
    x, y = 3.0 * np.sort(rng.random(n)) + 1.0, np.sort(rng.random(m)) - 2.0
    p, q = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
    T = (rng.exponential(size=(n, m)) / (n * m)).astype(np.float32)
    T64 = T.astype(np.float64)
    mom = (T64.sum(1), T64 @ y, T64.sum(0), x @ T64)
    Td = _to_dev(gw, T)
    Go = O.grad_prescribed(x, y, p, q, T64)
    G0 = gw.grad(x, y, p, q, Td).cpu().numpy().astype(np.float64)
    G1 = gw.grad(x, y, p, q, Td, moments=mom).cpu().numpy().astype(np.float64)
    assert _grad_err(G0, Go) <= GRAD_TOL and _grad_err(G1, Go) <= GRAD_TOL
    assert np.max(np.abs(G1 - G0)) <= 1e-6 * np.max(np.abs(Go))
    bad = (mom[0] * (1 + 1e-3), mom[1], mom[2], mom[3])
    G2 = gw.grad(x, y, p, q, Td, moments=bad).cpu().numpy().astype(np.float64)
    assert _grad_err(G2, Go) > 10 * GRAD_TOL
    from paper_2404_08970_b200 import _lib as L
    lib = L.load()
    z = torch.zeros(1, dtype=torch.float64, device=Td.device)
    mm = L.gw_moments(z.data_ptr(), None, z.data_ptr(), z.data_ptr())
    st = lib.gw_grad_dp(None, None, None, 0, None, 0, None)
    assert L.STATUS[st] == "GW_ERR_INVALID_ARG"
    with pytest.raises(GwError) as e:
        gw.grad(x, y, p, q, Td, moments=mom, k=2)
    assert e.value.code == "GW_ERR_UNSUPPORTED"
    del mm


def test_grad_deterministic(gw):
    P = W.config3(1500)
    Td = _to_dev(gw, P.extra["T"])
    a = gw.grad(P.x, P.y, P.p, P.q, Td).cpu().numpy()
    b = gw.grad(P.x, P.y, P.p, P.q, Td).cpu().numpy()
    assert np.array_equal(a, b)


# ----------------------------------------------------------------------------- errors

def test_rejects_unsorted(gw):
    from paper_2404_08970_b200 import GwError
    x = np.array([0.0, 0.5, 0.2, 0.9])
    T = np.full((4, 4), 1 / 16, np.float32)
    with pytest.raises(GwError) as e:
        gw.grad(x, np.sort(x), np.full(4, .25), np.full(4, .25), _to_dev(gw, T))
    assert e.value.code == "GW_ERR_UNSORTED"


def test_rejects_bad_marginals(gw):
    from paper_2404_08970_b200 import GwError
    x = np.linspace(0, 1, 4)
    T = _to_dev(gw, np.full((4, 4), 1 / 16, np.float32))
    with pytest.raises(GwError) as e:
        gw.grad(x, x, np.ones(4), np.full(4, .25), T)
    assert e.value.code == "GW_ERR_NOT_NORMALIZED"
    with pytest.raises(GwError) as e:
        gw.grad(x, x, np.array([.5, .5, .25, -.25]), np.full(4, .25), T)
    assert e.value.code == "GW_ERR_NEGATIVE_WEIGHT"
    # within the 1e-9 band: accepted (renormalised copy)
    gw.grad(x, x, np.array([.25, .25, .25, .25 + 1e-12]), np.full(4, .25), T)


# ----------------------------------------------------------------------------- Sinkhorn

@pytest.mark.parametrize("n,m,eps", [(5, 3, 0.2), (200, 333, 0.05), (1000, 2500, 0.02), (300, 4100, 0.01)])
def test_sinkhorn_parity(gw, n, m, eps):
    """sinkhorn_solve vs the oracle's log-domain Sinkhorn (same schedule, same fp32 cost)."""
    rng = np.random.default_rng(n + m)
    G = rng.random((n, m)).astype(np.float32)
    p, q = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
    r = gw.sinkhorn(_to_dev(gw, G), p, q, eps, 50, return_plan=True)
    f, g, _ = O.sinkhorn(G.astype(np.float64), p, q, eps, 50)
    To = O.plan_from_duals(G.astype(np.float64), f, g, eps)
    T = r["T"].cpu().numpy().astype(np.float64)
    eT = np.max(np.abs(T - To)) / np.max(To)
    eg = np.max(np.abs(r["g"].cpu().numpy() - g)) / eps
    print("sinkhorn_parity n=%d m=%d eps=%g: plan err/max T %.3e, dual err/eps %.3e" % (n, m, eps, eT, eg))
    assert eT <= PLAN_TOL and eg <= DUAL_TOL


def test_sinkhorn_tolerance_rule(gw):
    rng = np.random.default_rng(7)
    n, m, eps = 400, 300, 0.05
    G = rng.random((n, m)).astype(np.float32)
    p, q = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
    # tol = 1e-8: above the fp32 noise floor of marginals up to ~0.02 (the contract bound is 1e-6)
    r = gw.sinkhorn(_to_dev(gw, G), p, q, eps, 2000, tol=1e-8, check_every=10)
    assert r["converged"] and r["iters"] % 10 == 0 and r["violation"] <= 1e-8
    f, g, used = O.sinkhorn(G.astype(np.float64), p, q, eps, r["iters"])
    To = O.plan_from_duals(G.astype(np.float64), f, g, eps)
    assert O.violation(To, p, q) <= 1e-8


# ----------------------------------------------------------------------------- solver

def test_solver_c1_trajectory(gw):
    """C1 (BASELINE configs[0]): N = M = 256, eps = 1e-2, 20 x 100, T0 = p q^T, full trajectory."""
    P = W.config1()
    r = gw.solve(P.x, P.y, P.p, P.q, P.eps, P.outer, P.inner, trace_objective=True, return_plan=True)
    ro = O.entropic_gw(P.x, P.y, P.p, P.q, P.eps, P.outer, P.inner)
    assert abs(r.gw_objective - ro["gw_objective"]) <= OBJ_TOL * abs(ro["gw_objective"])
    assert r.marginal_violation <= VIOL_TOL
    np.testing.assert_allclose(r.trace[:, 0], ro["E"], rtol=OBJ_TOL)
    T = r.T.cpu().numpy().astype(np.float64)
    assert O.violation(T, P.p, P.q) <= VIOL_TOL
    assert abs(O.objective(P.x, P.y, T) - r.gw_objective) <= OBJ_TOL * abs(r.gw_objective)
    assert abs(r.entropic_objective - ro["entropic_objective"]) <= OBJ_TOL * abs(ro["entropic_objective"])


def test_solver_gradient_step_on_own_plan(gw):
    """The per-step gradient contract: c3 on the GPU's own T^l."""
    P = W.config2(1024)
    r = gw.solve(P.x, P.y, P.p, P.q, P.eps, 3, 100, return_plan=True)
    T = r.T
    G = gw.grad(P.x, P.y, P.p, P.q, T).cpu().numpy().astype(np.float64)
    Go = O.grad_prescribed(P.x, P.y, P.p, P.q, T.cpu().numpy().astype(np.float64))
    assert _grad_err(G, Go) <= GRAD_TOL


def test_solver_c2_recipe_reduced(gw):
    """C2 recipe at N = 1024 (Gaussian mixture / reflected y / Dirichlet marginals), eps = 5e-3,
    20 outer x 100 inner; the oracle replays the same schedule."""
    P = W.config2(1024)
    r = gw.solve(P.x, P.y, P.p, P.q, P.eps, 20, 100, trace_objective=True)
    ro = O.entropic_gw(P.x, P.y, P.p, P.q, P.eps, 20, 100)
    assert abs(r.gw_objective - ro["gw_objective"]) <= OBJ_TOL * abs(ro["gw_objective"])
    assert r.marginal_violation <= VIOL_TOL


def test_solver_tolerance_rule_replay(gw):
    """Reading R8: with the tolerance rule the GPU reports its per-outer inner counts and the
    oracle replays them exactly."""
    P = W.config4(512)
    r = gw.solve(P.x, P.y, P.p, P.q, P.eps, 5, 2000, tol=1e-7, check_every=10)
    counts = [int(c) for c in r.trace[:, 2]]
    ro = O.entropic_gw(P.x, P.y, P.p, P.q, P.eps, 5, counts)
    assert abs(r.gw_objective - ro["gw_objective"]) <= OBJ_TOL * abs(ro["gw_objective"])
    assert r.marginal_violation <= VIOL_TOL
    assert ro["viol"][-1] <= VIOL_TOL


def test_solver_single_point_and_row(gw):
    r = gw.solve([0.3], [0.7], [1.0], [1.0], 0.01, 3, 10, return_plan=True)
    assert r.T.cpu().numpy().tolist() == [[1.0]] and abs(r.gw_objective) < 1e-12
    rng = np.random.default_rng(1)
    y = np.sort(rng.random(9))
    q = rng.dirichlet(np.ones(9))
    r = gw.solve([0.5], y, [1.0], q, 0.01, 2, 20, return_plan=True)
    np.testing.assert_allclose(r.T.cpu().numpy()[0], q, rtol=1e-5)


def test_solver_host_vectors_match_device(gw):
    P = W.config1()
    a = gw.solve(P.x, P.y, P.p, P.q, P.eps, 4, 50)
    b = gw.solve_host(P.x, P.y, P.p, P.q, P.eps, 4, 50)
    assert a.gw_objective == b.gw_objective
    np.testing.assert_array_equal(a.f.cpu().numpy(), b.f)


def test_solver_deterministic(gw):
    P = W.config2(700)
    a = gw.solve(P.x, P.y, P.p, P.q, P.eps, 3, 60, return_plan=True)
    b = gw.solve(P.x, P.y, P.p, P.q, P.eps, 3, 60, return_plan=True)
    assert a.gw_objective == b.gw_objective
    assert np.array_equal(a.T.cpu().numpy(), b.T.cpu().numpy())


def test_ugw_argument_errors(gw):
    from paper_2404_08970_b200 import GwError
    P = W.config1()
    for kw, code in [({"rho": -1.0}, "GW_ERR_CONFIG"), ({"rho": float("inf")}, "GW_ERR_CONFIG"),
                     ({"eps": 0.0}, "GW_ERR_CONFIG")]:
        args = dict(rho=1.0, eps=0.01)
        args.update(kw)
        with pytest.raises(GwError) as e:
            gw.ugw_solve(P.x, P.y, P.p, P.q, args["rho"], args["eps"], 2, 10, device=_dev())
        assert e.value.code == code


# ----------------------------------------------------------------------------- fused path

@pytest.mark.parametrize("n,m,eps", [(300, 20000, 0.02), (64, 65536, 0.01), (500, 3000, 0.02), (257, 8193, 0.02),
                                     (1000, 8192, 0.01), (3, 70, 0.05), (200, 24576, 0.02), (150, 40001, 0.02)])
def test_sinkhorn_fused_path_parity(gw, monkeypatch, n, m, eps):
    """The fused one-read iteration (clusters of 1-8 CTAs spanning a row, ragged last CTA,
    CTAs entirely past m) against the oracle; and it must actually have run (the cluster-resident
    small path, which would take the small shapes, is switched off)."""
    monkeypatch.setenv("GWDP_NO_SMALL", "1")
    rng = np.random.default_rng(n * 7 + m)
    G = rng.random((n, m)).astype(np.float32)
    p, q = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
    r = gw.sinkhorn(_to_dev(gw, G), p, q, eps, 60, return_plan=True)
    assert r["fused_iters"] > 0
    f, g, _ = O.sinkhorn(G.astype(np.float64), p, q, eps, 60)
    To = O.plan_from_duals(G.astype(np.float64), f, g, eps)
    T = r["T"].cpu().numpy().astype(np.float64)
    eT = np.max(np.abs(T - To)) / np.max(To)
    print("fused_path_parity n=%d m=%d eps=%g: plan err/max T %.3e" % (n, m, eps, eT))
    assert eT <= PLAN_TOL


def test_fused_matches_safe_path(gw, monkeypatch):
    rng = np.random.default_rng(11)
    n, m, eps = 700, 12000, 0.02
    G = rng.random((n, m)).astype(np.float32)
    p, q = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
    Gd = _to_dev(gw, G)
    a = gw.sinkhorn(Gd, p, q, eps, 80)
    monkeypatch.setenv("GWDP_NO_FUSED", "1")
    b = gw.sinkhorn(Gd, p, q, eps, 80)
    assert a["fused_iters"] > 0 and b["fused_iters"] == 0
    # both are fp32-exponent evaluations of the same iteration: agree to the oracle tolerance
    np.testing.assert_allclose(a["g"].cpu().numpy(), b["g"].cpu().numpy(), rtol=0, atol=1e-4 * eps)
    np.testing.assert_allclose(a["f"].cpu().numpy(), b["f"].cpu().numpy(), rtol=0, atol=1e-4 * eps)


def test_solver_uses_fused_path(gw):
    P = W.config2(2048)
    r = gw.solve(P.x, P.y, P.p, P.q, P.eps, 4, 100)
    assert r.inner_fused_total > 200
    ro = O.entropic_gw(P.x, P.y, P.p, P.q, P.eps, 4, 100)
    assert abs(r.gw_objective - ro["gw_objective"]) <= OBJ_TOL * abs(ro["gw_objective"])


# ----------------------------------------------------------------------------- FGW (Remark 2)

def _c5_small(n=512, m=384, outer=5, inner=100):
    P = W.config5(n, m)
    P.outer, P.inner = outer, inner
    return P


@pytest.mark.parametrize("alpha", [0.5, 0.0, 1.0])
def test_fgw_solver_c5_recipe_reduced(gw, alpha):
    """fgw_solve vs oracle.entropic_fgw (reading R29) on C5's distributions at
    a reduced size: objective trajectory and final violation."""
    P = _c5_small()
    r = gw.solve(P.x, P.y, P.p, P.q, P.eps, P.outer, P.inner, fx=P.fx, fy=P.fy, alpha=alpha,
                 trace_objective=True, device=_dev())
    ro = O.entropic_fgw(P.x, P.y, P.p, P.q, P.fx, P.fy, alpha, P.eps, P.outer, P.inner)
    E = np.asarray(ro["E"])
    assert np.max(np.abs(r.trace[:, 0] - E) / np.abs(E)) <= OBJ_TOL
    assert abs(r.gw_objective - ro["gw_objective"]) <= OBJ_TOL * abs(ro["gw_objective"])
    assert r.marginal_violation <= max(VIOL_TOL, 2 * ro["viol"][-1])


def test_fgw_alpha_one_is_gw(gw):
    """alpha = 1 reduces FGW to GW (Remark 2): same trajectory as entropic_gw_solve."""
    P = _c5_small(300, 256, 4, 60)
    a = gw.solve(P.x, P.y, P.p, P.q, P.eps, P.outer, P.inner, fx=P.fx, fy=P.fy, alpha=1.0, device=_dev())
    b = gw.solve(P.x, P.y, P.p, P.q, P.eps, P.outer, P.inner, device=_dev())
    assert abs(a.gw_objective - b.gw_objective) <= 1e-6 * abs(b.gw_objective)


# ----------------------------------------------------------------------------- full-size configs

@pytest.mark.slow
def test_grad_c3_fullsize_full_matrix(gw):
    """C3 (BASELINE configs[2]) at its full size N = M = 16384: the whole gradient matrix against
    the dense definition (two float64 DGEMMs)."""
    P = W.config3(16384)
    T = P.extra["T"]
    G = gw.grad(P.x, P.y, P.p, P.q, _to_dev(gw, T)).cpu().numpy()
    Go = O.grad_prescribed(P.x, P.y, P.p, P.q, T.astype(np.float64))
    err = np.max(np.abs(G.astype(np.float64) - Go)) / np.max(np.abs(Go))
    assert err <= GRAD_TOL, err


@pytest.mark.slow
def test_solver_c2_fullsize_trajectory(gw):
    """C2 (BASELINE configs[1]) at its full size N = M = 4096, 20 outer x 100 inner: the GPU's
    objective trajectory against the oracle's (tests/golden/c2_n4096_trajectory.json, written
    by scripts/make_golden.py from oracle/ only)."""
    import json
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "c2_n4096_trajectory.json")
    ref = json.load(open(path))
    P = W.config2(4096)
    r = gw.solve(P.x, P.y, P.p, P.q, P.eps, 20, 100, trace_objective=True, device=_dev())
    E = np.asarray(ref["E"])
    assert np.max(np.abs(r.trace[:, 0] - E) / np.abs(E)) <= OBJ_TOL
    assert abs(r.gw_objective - ref["gw_objective"]) <= OBJ_TOL * abs(ref["gw_objective"])
    assert r.marginal_violation <= max(VIOL_TOL, 2 * ref["viol"][-1])


@pytest.mark.slow
def test_solver_c4_recipe_16384_trajectory(gw):
    """SURVEY §8(c) C4 parity (i): C4's recipe (eps = 1e-3, K = 100 fixed, 10 outer) at N = M = 16384,
    the GPU's objective trajectory against the oracle's (tests/golden/c4_n16384_trajectory.json,
    written by scripts/make_golden.py from oracle/ only)."""
    import json
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "c4_n16384_trajectory.json")
    if not os.path.exists(path):
        pytest.skip("golden trajectory not generated (python scripts/make_golden.py c4_16384)")
    ref = json.load(open(path))
    P = W.config4(16384)
    r = gw.solve(P.x, P.y, P.p, P.q, P.eps, 10, 100, trace_objective=True, device=_dev())
    E = np.asarray(ref["E"])
    assert np.max(np.abs(r.trace[:, 0] - E) / np.abs(E)) <= OBJ_TOL
    assert abs(r.gw_objective - ref["gw_objective"]) <= OBJ_TOL * abs(ref["gw_objective"])
    assert r.marginal_violation <= max(VIOL_TOL, 2 * ref["viol"][-1])


# ----------------------------------------------------------------------------- distance power k = 2 (f2)

@pytest.mark.parametrize("n,m", [(1, 5), (64, 64), (300, 517), (1024, 777)])
def test_grad_k2_random_plan(gw, n, m):
    """gw_grad_dp at k = 2 (D = |x - x'|^2) vs grad_prescribed(k=2)."""
    rng = np.random.default_rng(n + 7 * m)
    x, y = np.sort(rng.random(n)), np.sort(rng.random(m))
    p, q = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
    T = (rng.random((n, m)) / (n * m)).astype(np.float32)
    G = gw.grad(x, y, p, q, _to_dev(gw, T), k=2).cpu().numpy().astype(np.float64)
    Go = O.grad_prescribed(x, y, p, q, T.astype(np.float64), k=2)
    assert _grad_err(G, Go) <= GRAD_TOL


def test_solver_k2_trajectory(gw):
    """Entropic GW at k = 2 on C5's distributions (reduced): objective trajectory vs the oracle."""
    P = _c5_small(400, 300, 5, 100)
    r = gw.solve(P.x, P.y, P.p, P.q, P.eps, P.outer, P.inner, trace_objective=True, device=_dev(), k=2)
    ro = O.entropic_gw(P.x, P.y, P.p, P.q, P.eps, P.outer, P.inner, k=2)
    E = np.asarray(ro["E"])
    assert np.max(np.abs(r.trace[:, 0] - E) / np.abs(E)) <= OBJ_TOL
    assert abs(r.gw_objective - ro["gw_objective"]) <= OBJ_TOL * abs(ro["gw_objective"])
    assert r.marginal_violation <= max(VIOL_TOL, 2 * ro["viol"][-1])


def test_fgw_k2(gw):
    P = _c5_small(300, 256, 4, 60)
    r = gw.solve(P.x, P.y, P.p, P.q, P.eps, P.outer, P.inner, fx=P.fx, fy=P.fy, alpha=0.5, device=_dev(), k=2)
    ro = O.entropic_fgw(P.x, P.y, P.p, P.q, P.fx, P.fy, 0.5, P.eps, P.outer, P.inner, k=2)
    assert abs(r.gw_objective - ro["gw_objective"]) <= OBJ_TOL * abs(ro["gw_objective"])


# ----------------------------------------------------------------------------- distance powers k = 3..5 (f2)

@pytest.mark.parametrize("k", [3, 4, 5])
@pytest.mark.parametrize("n,m", [(1, 1), (1, 9), (7, 1), (128, 128), (129, 257), (300, 517), (1000, 777)])
def test_grad_kgen_random_plan(gw, k, n, m):
    """gw_grad_dp at k = 3..5 (D = |x - x'|^k) vs grad_prescribed(k):
    tiles of 128 with ragged tails, ties, non-uniform marginals."""
    rng = np.random.default_rng(13 * n + m + k)
    x, y = np.sort(rng.random(n)), np.sort(rng.random(m))
    if n > 10:
        x[5] = x[4]
    p, q = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
    T = (rng.exponential(size=(n, m)) / (n * m)).astype(np.float32)
    G = gw.grad(x, y, p, q, _to_dev(gw, T), k=k).cpu().numpy().astype(np.float64)
    Go = O.grad_prescribed(x, y, p, q, T.astype(np.float64), k=k)
    assert _grad_err(G, Go) <= GRAD_TOL


@pytest.mark.parametrize("k", [3, 5])
@pytest.mark.parametrize("shape", ["wide", "clustered", "long"])
def test_grad_kgen_tile_centred_fp32(gw, k, shape):
    """k = 3, 5 run fp32 arithmetic about each 128-wide tile's own centre, with fp64 carries between
    tiles (polyk.cuh): wide shifted supports, a tight cluster holding most of the mass beside far
    outliers (a big carry next to small local terms), and long rows (64 column tiles' carries summed
    into one row) -- each against the dense definition at the gradient tolerance."""
    rng = np.random.default_rng(100 * k + len(shape))
    if shape == "wide":
        n, m = 1500, 1300
        x, y = 10.0 * np.sort(rng.random(n)) - 3.0, 4.0 * np.sort(rng.random(m)) + 1.0
    elif shape == "clustered":
        n, m = 1100, 900
        x = np.sort(np.concatenate([0.5 + 1e-3 * rng.random(n - 20), rng.random(20) * 3.0 - 1.0]))
        y = np.sort(np.concatenate([0.2 + 1e-3 * rng.random(m - 10), rng.random(10) * 2.0]))
    else:
        n, m = 300, 8192
        x, y = np.sort(rng.random(n)), np.sort(rng.random(m))
    p, q = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
    T = (rng.exponential(size=(n, m)) / (n * m)).astype(np.float32)
    G = gw.grad(x, y, p, q, _to_dev(gw, T), k=k).cpu().numpy().astype(np.float64)
    Go = O.grad_prescribed(x, y, p, q, T.astype(np.float64), k=k)
    err = _grad_err(G, Go)
    print("k=%d %s n=%d m=%d: gradient err / max|G| %.3e" % (k, shape, n, m, err))
    assert err <= GRAD_TOL


@pytest.mark.parametrize("n,m", [(2048, 2048), (1500, 16384)])
def test_grad_k4_moments_path(gw, n, m):
    """k = 4 runs the polynomial-moments path (poly.cuh: 25 plan moments + an fp64 degree-4 polynomial
    per row; 4NM + 4NM bytes): wide, shifted supports and long rows (fp32 partial moment sums over many
    columns) against the dense definition."""
    rng = np.random.default_rng(n + m)
    x, y = 10.0 * np.sort(rng.random(n)) - 3.0, 4.0 * np.sort(rng.random(m)) + 1.0
    p, q = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
    T = (rng.exponential(size=(n, m)) / (n * m)).astype(np.float32)
    G = gw.grad(x, y, p, q, _to_dev(gw, T), k=4).cpu().numpy().astype(np.float64)
    Go = O.grad_prescribed(x, y, p, q, T.astype(np.float64), k=4)
    err = _grad_err(G, Go)
    print("k=4 moments path n=%d m=%d: gradient err / max|G| %.3e" % (n, m, err))
    assert err <= GRAD_TOL


def test_grad_k3_c3_recipe_2048(gw):
    """k = 3 on the C3 recipe (Exp(1) plan rescaled to uniform marginals), wide supports."""
    P = W.config3(2048)
    T = P.extra["T"]
    x, y = 10.0 * P.x - 3.0, 4.0 * P.y + 1.0
    G = gw.grad(x, y, P.p, P.q, _to_dev(gw, T), k=3).cpu().numpy().astype(np.float64)
    Go = O.grad_prescribed(x, y, P.p, P.q, T.astype(np.float64), k=3)
    assert _grad_err(G, Go) <= GRAD_TOL


@pytest.mark.parametrize("k", [3, 4])
def test_solver_kgen_trajectory(gw, k):
    """Entropic GW at k = 3, 4 on C5's distributions (reduced): objective trajectory vs the oracle."""
    P = _c5_small(400, 300, 5, 100)
    r = gw.solve(P.x, P.y, P.p, P.q, P.eps, P.outer, P.inner, trace_objective=True, device=_dev(), k=k)
    ro = O.entropic_gw(P.x, P.y, P.p, P.q, P.eps, P.outer, P.inner, k=k)
    E = np.asarray(ro["E"])
    assert np.max(np.abs(r.trace[:, 0] - E) / np.abs(E)) <= OBJ_TOL
    assert abs(r.gw_objective - ro["gw_objective"]) <= OBJ_TOL * abs(ro["gw_objective"])
    assert abs(r.entropic_objective - ro["entropic_objective"]) <= OBJ_TOL * abs(ro["entropic_objective"])
    assert r.marginal_violation <= max(VIOL_TOL, 2 * ro["viol"][-1])


def test_fgw_k3(gw):
    P = _c5_small(300, 256, 4, 60)
    r = gw.solve(P.x, P.y, P.p, P.q, P.eps, P.outer, P.inner, fx=P.fx, fy=P.fy, alpha=0.5, device=_dev(), k=3)
    ro = O.entropic_fgw(P.x, P.y, P.p, P.q, P.fx, P.fy, 0.5, P.eps, P.outer, P.inner, k=3)
    assert abs(r.gw_objective - ro["gw_objective"]) <= OBJ_TOL * abs(ro["gw_objective"])


def test_k6_unsupported(gw):
    from paper_2404_08970_b200 import GwError
    rng = np.random.default_rng(0)
    x = np.sort(rng.random(16))
    p = np.full(16, 1 / 16)
    T = _to_dev(gw, np.full((16, 16), 1 / 256, dtype=np.float32))
    for k in (0, 6):
        with pytest.raises(GwError) as e:
            gw.grad(x, x, p, p, T, k=k)
        assert e.value.code == "GW_ERR_UNSUPPORTED"


# ----------------------------------------------------------------------------- tau != eps (Remark 1)

@pytest.mark.parametrize("tau_ratio", [0.5, 2.0])
def test_solver_general_tau(gw, tau_ratio):
    """PAPER.md:102-110 with tau != eps: cost grad E + (eps - tau) ln T^l at regulariser tau, vs
    oracle.entropic_gw(tau=...) (pinned against the KL-proximal step)."""
    P = _c5_small(400, 300, 5, 100)
    tau = tau_ratio * P.eps
    r = gw.solve(P.x, P.y, P.p, P.q, P.eps, P.outer, P.inner, trace_objective=True, device=_dev(), tau=tau)
    ro = O.entropic_gw(P.x, P.y, P.p, P.q, P.eps, P.outer, P.inner, tau=tau)
    E = np.asarray(ro["E"])
    assert np.max(np.abs(r.trace[:, 0] - E) / np.abs(E)) <= OBJ_TOL
    assert abs(r.gw_objective - ro["gw_objective"]) <= OBJ_TOL * abs(ro["gw_objective"])
    assert abs(r.entropic_objective - ro["entropic_objective"]) <= OBJ_TOL * abs(ro["entropic_objective"])
    assert r.marginal_violation <= max(VIOL_TOL, 2 * ro["viol"][-1])


def test_general_tau_fgw_and_unsupported(gw):
    from paper_2404_08970_b200 import GwError
    P = _c5_small(300, 256, 3, 60)
    r = gw.solve(P.x, P.y, P.p, P.q, P.eps, P.outer, P.inner, fx=P.fx, fy=P.fy, alpha=0.5, device=_dev(),
                 tau=0.5 * P.eps)
    ro = O.entropic_fgw(P.x, P.y, P.p, P.q, P.fx, P.fy, 0.5, P.eps, P.outer, P.inner, tau=0.5 * P.eps)
    assert abs(r.gw_objective - ro["gw_objective"]) <= OBJ_TOL * abs(ro["gw_objective"])
    with pytest.raises(GwError) as e:
        gw.solve(P.x, P.y, P.p, P.q, P.eps, 2, 10, device=_dev(), tau=0.5 * P.eps, k=2)
    assert e.value.code == "GW_ERR_UNSUPPORTED"


# ----------------------------------------------------------------------------- cluster-resident small path

@pytest.mark.parametrize("n,m", [(256, 256), (400, 300), (37, 1000), (1, 9)])
def test_small_cluster_path_matches_multikernel_path(gw, monkeypatch, n, m):
    """small.cuh (one launch per inner loop, G in one cluster's shared memory) against the
    multi-kernel path and the oracle on the same problem."""
    rng = np.random.default_rng(n + m)
    x, y = np.sort(rng.random(n)), np.sort(rng.random(m))
    p, q = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
    eps = 0.02
    a = gw.solve(x, y, p, q, eps, 4, 80, trace_objective=True, device=_dev())
    monkeypatch.setenv("GWDP_NO_SMALL", "1")
    b = gw.solve(x, y, p, q, eps, 4, 80, trace_objective=True, device=_dev())
    monkeypatch.delenv("GWDP_NO_SMALL")
    ro = O.entropic_gw(x, y, p, q, eps, 4, 80)
    E = np.asarray(ro["E"])
    for r in (a, b):
        assert np.max(np.abs(r.trace[:, 0] - E) / np.abs(E)) <= OBJ_TOL
        assert r.marginal_violation <= max(VIOL_TOL, 2 * ro["viol"][-1])
    # two fp32 evaluations of the same schedule (fp64 small-path exponents vs the fused path's fp32 ones):
    # each is within 1e-4 of the oracle above; between them, 3e-5
    assert abs(a.gw_objective - b.gw_objective) <= 3e-5 * abs(b.gw_objective)


# ----------------------------------------------------------------------------- fault injection

def test_fault_injection_is_caught(gw, monkeypatch):
    """A test-only hook perturbs one tile carry of the gradient (GWDP_FAULT=carry) or one column sum
    of the fused Sinkhorn iteration (GWDP_FAULT=colsum) by a factor 2: the parity checks must fail."""
    rng = np.random.default_rng(5)
    n, m = 600, 700
    x, y = np.sort(rng.random(n)), np.sort(rng.random(m))
    p, q = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
    T = (rng.random((n, m)) / (n * m)).astype(np.float32)
    Go = O.grad_prescribed(x, y, p, q, T.astype(np.float64))
    G = gw.grad(x, y, p, q, _to_dev(gw, T)).cpu().numpy().astype(np.float64)
    assert _grad_err(G, Go) <= GRAD_TOL
    monkeypatch.setenv("GWDP_FAULT", "carry")
    Gf = gw.grad(x, y, p, q, _to_dev(gw, T)).cpu().numpy().astype(np.float64)
    assert _grad_err(Gf, Go) > GRAD_TOL
    monkeypatch.setenv("GWDP_FAULT", "colsum")
    monkeypatch.setenv("GWDP_NO_SMALL", "1")
    Gc = rng.random((300, 20000)).astype(np.float32)
    pc, qc = rng.dirichlet(np.ones(300)), rng.dirichlet(np.ones(20000))
    r = gw.sinkhorn(_to_dev(gw, Gc), pc, qc, 0.02, 60, return_plan=True)
    f, g, _ = O.sinkhorn(Gc.astype(np.float64), pc, qc, 0.02, 60)
    To = O.plan_from_duals(Gc.astype(np.float64), f, g, 0.02)
    assert r["fused_iters"] > 0
    assert np.max(np.abs(r["T"].cpu().numpy().astype(np.float64) - To)) > 1e-4 * np.max(To)


def test_general_tau_degenerate_shapes(gw):
    r = gw.solve([0.3], [0.7], [1.0], [1.0], 0.02, 3, 10, tau=0.01, return_plan=True, device=_dev())
    assert r.T.cpu().numpy().tolist() == [[1.0]] and abs(r.gw_objective) < 1e-12


# ----------------------------------------------------------------------------- regression (round-1 advice)

def test_solver_zero_outer_with_T0_returns_T0(gw):
    """outer_iters == 0 with an explicit T0 and a returned plan: the plan IS T0 and the objective is
    E(T0) (no Gibbs regeneration from absent duals)."""
    rng = np.random.default_rng(11)
    n, m = 40, 33
    x, y = np.sort(rng.random(n)), np.sort(rng.random(m))
    p, q = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
    T0 = (np.outer(p, q) * rng.uniform(0.5, 1.5, (n, m))).astype(np.float32)
    r = gw.solve(x, y, p, q, 0.05, 0, 10, T0=_to_dev(gw, T0), return_plan=True)
    assert np.array_equal(r.T.cpu().numpy(), T0)
    Eo = O.objective(x, y, T0.astype(np.float64))
    assert abs(r.gw_objective - Eo) <= 1e-5 * abs(Eo)


def test_solver_tolerance_early_stop_consistent_plan(gw):
    """tol > 0 with an early stop: the measuring row half-step splits a DISCARDED trial f' into the
    fp32 dual parts; they must be re-split from the committed f, so that the reported objective and
    violation (computed from the fp32 parts) describe the returned plan and duals (computed from f).
    With and without the objective trace (which runs the fp64-regeneration gradient kernels) the
    schedules agree and the results agree to the fp32 tolerance."""
    P = W.config2(512)
    a = gw.solve(P.x, P.y, P.p, P.q, 2e-2, 4, 2000, tol=1e-6, check_every=10, return_plan=True)
    b = gw.solve(P.x, P.y, P.p, P.q, 2e-2, 4, 2000, tol=1e-6, check_every=10, trace_objective=True,
                 return_plan=True)
    assert list(a.trace[:, 2]) == list(b.trace[:, 2])
    assert int(a.trace[-1, 2]) < 2000  # the early stop happened
    for r in (a, b):
        T = r.T.cpu().numpy().astype(np.float64)
        Eo = O.objective(P.x, P.y, T)
        assert abs(r.gw_objective - Eo) <= 1e-5 * abs(Eo)
        vo = O.violation(T, P.p, P.q)
        assert abs(r.marginal_violation - vo) <= 2e-8 + 0.05 * vo
    np.testing.assert_allclose(a.f.cpu().numpy(), b.f.cpu().numpy(), rtol=0, atol=1e-4 * 2e-2)
    counts = [int(c) for c in a.trace[:, 2]]
    ro = O.entropic_gw(P.x, P.y, P.p, P.q, 2e-2, 4, counts)
    assert abs(a.gw_objective - ro["gw_objective"]) <= OBJ_TOL * abs(ro["gw_objective"])


def test_single_rank_rejects_partial_shard(gw):
    """One rank: (row0, n_local) must be (0, n); a partial shard would silently drop rows."""
    from paper_2404_08970_b200 import GwError
    rng = np.random.default_rng(3)
    x = np.sort(rng.random(64))
    p = np.full(64, 1.0 / 64)
    for row0, nl in [(0, 32), (16, 48)]:
        with pytest.raises(GwError) as e:
            gw.solve(x, x, p, p, 0.1, 1, 5, row0=row0, n_local=nl, device=_dev())
        assert e.value.code == "GW_ERR_DIM_MISMATCH"
    with pytest.raises(GwError):  # an empty shard (null f) is rejected before any work
        gw.solve(x, x, p, p, 0.1, 1, 5, row0=0, n_local=0, device=_dev())
