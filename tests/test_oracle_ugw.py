"""Pins for the UGW oracle (oracle/ugw.py; Remark 3; readings R32-R35).
The paper leaves g(G^) undefined; these tests pin every piece of the reading to something other
than itself and the whole loop by its fixed point (a critical point of the functional Remark 3
minimises).  The per-iteration trajectory has no worked example in the paper: parity unpinned."""

import math

import numpy as np
import pytest

import oracle as O


def _problem(seed, n, m):
    rng = np.random.default_rng(seed)
    x, y = np.sort(rng.random(n)), np.sort(rng.random(m))
    u, v = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
    return rng, x, y, u, v


def test_kl_tensor_closed_form_is_bruteforce():
    rng = np.random.default_rng(0)
    a, b = rng.random(5) * 0.3, rng.random(5) * 0.4
    assert abs(O.kl_tensor_sq(a, b) - O.kl(np.outer(a, a), np.outer(b, b))) <= 1e-13
    assert O.kl(b, b) == pytest.approx(0.0, abs=1e-15)


def test_functional_closed_form_is_bruteforce():
    rng, x, y, u, v = _problem(1, 4, 3)
    G = rng.random((4, 3)) * 0.1
    for k in (1, 2):
        a = O.ugw_functional(x, y, u, v, G, 0.7, 0.05, k)
        b = O.ugw_functional_bruteforce(x, y, u, v, G, 0.7, 0.05, k)
        assert abs(a - b) <= 1e-12 * max(1.0, abs(b))


@pytest.mark.parametrize("k,su,sv", [(1, 1.0, 1.0), (2, 1.0, 1.0), (1, 0.6, 1.7)])
def test_ugw_cost_is_half_gradient_of_functional(k, su, sv):
    """R32: the subproblem's linearised objective L(G) = <C(G^), G> + m(G^) (rho KL(G1|u) +
    rho KL(G^T1|v) + eps KL(G|uv)) has gradient 1/2 grad F_eps at G = G^ (F_eps brute force,
    central differences): this fixes g(G^) and the realised-marginal 1/2 grad E.  Also for
    measures u, v of mass != 1 (unbalanced inputs)."""
    rng, x, y, u, v = _problem(2 + k, 4, 3)
    u, v = su * u, sv * v
    Gh = rng.random((4, 3)) * 0.15 + 0.01
    rho, eps = 0.8, 0.07
    C = O.ugw_cost(x, y, u, v, Gh, rho, eps, k)
    a, b = Gh.sum(1), Gh.sum(0)
    mh = Gh.sum()
    gradL = C + mh * (rho * np.log(a / u)[:, None] + rho * np.log(b / v)[None, :] + eps * np.log(Gh / np.outer(u, v)))
    h = 1e-6
    for _ in range(3):
        D = rng.standard_normal(Gh.shape)
        fp = O.ugw_functional_bruteforce(x, y, u, v, Gh + h * D, rho, eps, k)
        fm = O.ugw_functional_bruteforce(x, y, u, v, Gh - h * D, rho, eps, k)
        fd = (fp - fm) / (2 * h)
        assert abs(fd - 2.0 * np.sum(gradL * D)) <= 1e-6 * max(1.0, abs(fd))


def test_unbalanced_sinkhorn_solves_the_primal():
    """R34: the converged unbalanced Sinkhorn plan minimises <C,G> + eps KL(G|uv) + rho KL(G1|u)
    + rho KL(G^T1|v) (direct L-BFGS minimisation of the primal over log G, tiny instance)."""
    from scipy.optimize import minimize
    rng = np.random.default_rng(7)
    n, m = 3, 4
    u, v = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m)) * 1.3
    C = rng.random((n, m))
    rho, eps = 0.6, 0.2
    f, g = O.unbalanced_sinkhorn(C, u, v, rho, eps, 3000)
    Gs = O.unbalanced_plan(C, u, v, f, g, eps)

    def primal(z):
        G = np.exp(z.reshape(n, m))
        a, b = G.sum(1), G.sum(0)
        val = np.sum(C * G) + eps * O.kl(G, np.outer(u, v)) + rho * O.kl(a, u) + rho * O.kl(b, v)
        dG = C + eps * np.log(G / np.outer(u, v)) + rho * np.log(a / u)[:, None] + rho * np.log(b / v)[None, :]
        return val, (dG * G).ravel()

    r = minimize(primal, np.log(np.outer(u, v)).ravel(), jac=True, method="L-BFGS-B",
                 options={"ftol": 1e-15, "gtol": 1e-13, "maxiter": 10000})
    Gp = np.exp(r.x.reshape(n, m))
    np.testing.assert_allclose(Gs, Gp, rtol=2e-5, atol=1e-9)
    assert primal(np.log(Gs).ravel())[0] <= r.fun + 1e-12


def test_ugw_balanced_limit_is_entropic_gw_at_twice_eps():
    """rho -> infinity: kappa -> 1, the subproblem is balanced entropic OT of 1/2 grad E at eps,
    i.e. of grad E at 2 eps (constants drop out); with converged inner loops the UGW iteration
    reproduces oracle.entropic_gw(eps = 2 eps) (R32-R35 at their balanced limit)."""
    _, x, y, u, v = _problem(11, 7, 6)
    eps = 0.05
    ru = O.entropic_ugw(x, y, u, v, 1e9, eps, 4, 3000)
    rg = O.entropic_gw(x, y, u, v, 2 * eps, 4, 3000)
    np.testing.assert_allclose(ru["E"], rg["E"], rtol=1e-7)
    np.testing.assert_allclose(ru["T"], rg["T"], atol=1e-9)
    assert abs(ru["mass"][-1] - 1.0) <= 1e-7


def test_ugw_mass_rescaling_and_symmetry():
    """R35: after each step m(G) = sqrt(m(G^) m(G_sinkhorn)); swapping the spaces transposes the
    plan (the functional is symmetric in X, Y)."""
    _, x, y, u, v = _problem(5, 6, 5)
    r1 = O.entropic_ugw(x, y, u, v, 0.5, 0.05, 3, 200)
    r2 = O.entropic_ugw(y, x, v, u, 0.5, 0.05, 3, 200)
    np.testing.assert_allclose(r1["F"], r2["F"], rtol=1e-10)
    assert all(0.0 < mm < 1.0 + 1e-9 for mm in r1["mass"])


@pytest.mark.parametrize("rho,eps", [(1.0, 0.1), (0.5, 0.05)])
def test_ugw_fixed_point_is_a_critical_point_of_the_functional(rho, eps):
    """Remark 3 minimises F_eps over all positive measures (no constraint), by
    alternate minimisation of the bi-convex relaxation; a fixed point G = G^ of the whole iteration
    (readings R32-R35: cost 1/2 grad E + g, the mass-scaled rho~, eps~, the square-root rescaling)
    therefore has grad F_eps(G) = 0 entrywise.  Checked by central differences of the BRUTE-FORCE
    functional; any mistake in the loop's scalings (rho~ = rho, no square root, a wrong g(G^)) moves
    the fixed point off the critical set.  Masses of u, v differ from 1 and from each other."""
    rng, x, y, u, v = _problem(3, 5, 4)
    u, v = 0.8 * u, 1.3 * v
    r = O.entropic_ugw(x, y, u, v, rho, eps, 300, 300)
    T = np.asarray(r["T"])
    assert abs(r["F"][-1] - r["F"][-2]) <= 1e-13

    def grad_fd(Z):
        g = np.zeros_like(Z)
        for i in range(Z.shape[0]):
            for j in range(Z.shape[1]):
                h = 1e-6 * Z[i, j]
                Zp, Zm = Z.copy(), Z.copy()
                Zp[i, j] += h
                Zm[i, j] -= h
                g[i, j] = (O.ugw_functional_bruteforce(x, y, u, v, Zp, rho, eps, 1)
                           - O.ugw_functional_bruteforce(x, y, u, v, Zm, rho, eps, 1)) / (2 * h)
        return g
    g0 = np.abs(grad_fd(np.outer(u, v) / math.sqrt(u.sum() * v.sum()))).max()
    assert g0 > 0.1                                   # the start plan is far from critical
    assert np.abs(grad_fd(T)).max() <= 1e-6 * g0      # measured 3e-8 / 0.35


def test_ugw_start_and_masses():
    """R35 for measures of any mass: the iteration starts from u v / sqrt(m(u) m(v)), so its first
    functional value is the brute-force F_eps of that plan after one step of mass balance, and the
    mass trajectory stays positive; scaling both u and v by the same s leaves the balanced-mass
    plan's realised marginals proportional to u and v at G^0 (checked on the start plan)."""
    _, x, y, u, v = _problem(7, 5, 4)
    u, v = 0.6 * u, 1.7 * v
    r0 = O.entropic_ugw(x, y, u, v, 0.5, 0.05, 0, 10)
    G0 = np.asarray(r0["T"])
    np.testing.assert_allclose(G0, np.outer(u, v) / math.sqrt(u.sum() * v.sum()), rtol=1e-15)
    np.testing.assert_allclose(G0.sum(), math.sqrt(u.sum() * v.sum()), rtol=1e-14)
    r = O.entropic_ugw(x, y, u, v, 0.5, 0.05, 2, 200)
    assert all(mm > 0.0 for mm in r["mass"])
    Fb = O.ugw_functional_bruteforce(x, y, u, v, r["T"], 0.5, 0.05, 1)
    assert abs(r["F"][-1] - Fb) <= 1e-12 * max(1.0, abs(Fb))
