"""GPU parity for entropic unbalanced GW (Remark 3, PAPER.md:148-167,
readings R32-R35): ugw_solve through the C ABI against oracle.entropic_ugw on the same seeded
inputs (C5's distributions at reduced sizes, rho = 1.0 as BASELINE's C5 names).  The reading
itself is parity unpinned (the paper leaves g undefined); the oracle's pieces are pinned in
tests/test_oracle_ugw.py."""

import numpy as np
import pytest

import oracle as O
import workloads as W

pytestmark = pytest.mark.gpu

OBJ_TOL = 1e-4


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


@pytest.mark.parametrize("n,m,rho,eps,k", [(300, 256, 1.0, 0.01, 1), (257, 129, 0.3, 0.02, 1),
                                           (200, 180, 1.0, 0.01, 2), (150, 160, 2.0, 0.02, 3)])
def test_ugw_trajectory(gw, n, m, rho, eps, k):
    P = W.config5(n, m)
    outer, inner = 5, 60
    r = gw.ugw_solve(P.x, P.y, P.p, P.q, rho, eps, outer, inner, trace_objective=True, return_plan=True,
                     device=_dev(), k=k)
    ro = O.entropic_ugw(P.x, P.y, P.p, P.q, rho, eps, outer, inner, k=k)
    F, E, mass = np.asarray(ro["F"]), np.asarray(ro["E"]), np.asarray(ro["mass"])
    assert np.max(np.abs(r.trace[:, 0] - F) / np.abs(F)) <= OBJ_TOL
    assert np.max(np.abs(r.trace[:, 1] - E) / np.abs(E)) <= OBJ_TOL
    np.testing.assert_allclose(r.trace[:, 3], mass, rtol=1e-5)
    assert abs(r.gw_objective - E[-1]) <= OBJ_TOL * abs(E[-1])
    assert abs(r.entropic_objective - F[-1]) <= OBJ_TOL * abs(F[-1])
    T = r.T.cpu().numpy().astype(np.float64)
    assert np.max(np.abs(T - ro["T"])) <= 1e-3 * np.max(ro["T"])
    assert abs(T.sum() - mass[-1]) <= 1e-5 * mass[-1]


def test_ugw_zero_outer_is_product(gw):
    P = W.config5(64, 48)
    r = gw.ugw_solve(P.x, P.y, P.p, P.q, 1.0, 0.01, 0, 10, return_plan=True, device=_dev())
    np.testing.assert_allclose(r.T.cpu().numpy(), np.outer(P.p, P.q), rtol=1e-6, atol=1e-12)
    assert abs(r.gw_objective - O.objective(P.x, P.y, np.outer(P.p, P.q))) <= 1e-6 * abs(r.gw_objective)
    assert abs(r.entropic_objective - r.gw_objective) <= 1e-9


def test_ugw_large_rho_approaches_balanced_gw(gw):
    """rho -> infinity (R32-R35): the UGW plan at rho = 1e6 is the balanced entropic GW plan at
    2 eps up to O(eps / rho) (both on the GPU; the oracle pins the exact limit)."""
    P = W.config5(200, 150)
    r = gw.ugw_solve(P.x, P.y, P.p, P.q, 1e6, 0.02, 4, 300, return_plan=True, device=_dev())
    b = gw.solve(P.x, P.y, P.p, P.q, 0.04, 4, 300, return_plan=True, device=_dev())
    assert abs(r.gw_objective - b.gw_objective) <= 1e-3 * abs(b.gw_objective)
    assert abs(r.trace[-1, 3] - 1.0) <= 1e-4


@pytest.mark.parametrize("n,m", [(1, 1), (1, 5), (6, 1)])
def test_ugw_degenerate_shapes(gw, n, m):
    """Single-point spaces: E = 0 (one row or column of a plan has no pair distances to mismatch);
    the iteration still runs and matches the oracle's mass trajectory."""
    rng = np.random.default_rng(n * 10 + m)
    x, y = np.sort(rng.random(n)), np.sort(rng.random(m))
    u, v = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
    r = gw.ugw_solve(x, y, u, v, 1.0, 0.05, 3, 30, trace_objective=True, device=_dev())
    ro = O.entropic_ugw(x, y, u, v, 1.0, 0.05, 3, 30)
    np.testing.assert_allclose(r.trace[:, 3], ro["mass"], rtol=1e-5)
    assert abs(r.entropic_objective - ro["F"][-1]) <= 1e-4 * max(abs(ro["F"][-1]), 1e-12)


@pytest.mark.parametrize("n,m,k,su,sv", [(300, 256, 1, 0.6, 1.7), (200, 180, 2, 2.5, 0.8), (150, 160, 3, 1.0, 0.4)])
def test_ugw_trajectory_unequal_masses(gw, n, m, k, su, sv):
    """Unbalanced inputs proper: u, v of masses != 1 (and != each other), G^0 = u v / sqrt(m(u) m(v))
    (R35), KL constants m(u)^2, m(v)^2, (m(u) m(v))^2 in F_eps (R33)."""
    P = W.config5(n, m)
    u, v = su * P.p, sv * P.q
    outer, inner = 4, 60
    r = gw.ugw_solve(P.x, P.y, u, v, 1.0, 0.01, outer, inner, trace_objective=True, return_plan=True,
                     device=_dev(), k=k)
    ro = O.entropic_ugw(P.x, P.y, u, v, 1.0, 0.01, outer, inner, k=k)
    F, E, mass = np.asarray(ro["F"]), np.asarray(ro["E"]), np.asarray(ro["mass"])
    assert np.max(np.abs(r.trace[:, 0] - F) / np.abs(F)) <= OBJ_TOL
    assert np.max(np.abs(r.trace[:, 1] - E) / np.abs(E)) <= OBJ_TOL
    np.testing.assert_allclose(r.trace[:, 3], mass, rtol=1e-5)
    T = r.T.cpu().numpy().astype(np.float64)
    assert np.max(np.abs(T - ro["T"])) <= 1e-3 * np.max(ro["T"])


def test_ugw_zero_outer_unequal_masses(gw):
    P = W.config5(64, 48)
    u, v = 0.5 * P.p, 3.0 * P.q
    r = gw.ugw_solve(P.x, P.y, u, v, 1.0, 0.01, 0, 10, return_plan=True, device=_dev())
    T0 = np.outer(u, v) / np.sqrt(u.sum() * v.sum())
    np.testing.assert_allclose(r.T.cpu().numpy(), T0, rtol=1e-6, atol=1e-12)
    assert abs(r.gw_objective - O.objective(P.x, P.y, T0)) <= 1e-6 * abs(r.gw_objective)
    Fo = O.ugw_functional(P.x, P.y, u, v, T0, 1.0, 0.01)
    assert abs(r.entropic_objective - Fo) <= 1e-6 * abs(Fo)


def test_ugw_rejects_zero_mass(gw):
    from paper_2404_08970_b200._lib import GwError
    P = W.config5(16, 12)
    with pytest.raises(GwError):
        gw.ugw_solve(P.x, P.y, np.zeros(16), P.q, 1.0, 0.01, 1, 5, device=_dev())
