"""Pins for the float64 oracle (-m "not gpu").

Each test ties an oracle function to something other than itself: worked
examples printed in SPEC.md/PAPER.md (tests/golden/), closed forms derived
independently here, brute force on tiny inputs, invariants, finite differences
and an independent convex solver.  A plausible mistake in the oracle (dropped
term, wrong sign or index, transposed operand, wrong factor 2 or 4, wrong
schedule) fails at least one of them.
"""

import itertools
import json
import math
import os

import numpy as np
import pytest

import oracle as O
import workloads as W

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def _sorted(rng, n):
    return np.sort(rng.random(n))


def _feasible_plan(rng, p, q, iters=2000):
    """A strictly positive plan in S(p, q), built by alternating rescaling of a random
    matrix (input preparation only, independent of the oracle's Sinkhorn)."""
    Z = rng.random((p.size, q.size)) + 0.1
    for _ in range(iters):
        Z *= (p / Z.sum(1))[:, None]
        Z *= (q / Z.sum(0))[None, :]
    return Z


# --------------------------------------------------------------------------- golden

@pytest.mark.parametrize("ex", GOLDEN["dp"], ids=lambda e: e["id"])
def test_dp_worked_examples(ex):
    fn = {"lower": O.ref_dp_lower, "upper": O.ref_dp_upper, "distance": O.ref_dp_distance}[ex["op"]]
    np.testing.assert_allclose(fn(ex["v"], ex["s"], ex["k"]), ex["expect"], rtol=0, atol=1e-14)


@pytest.mark.parametrize("ex", GOLDEN["dist"], ids=lambda e: e["id"])
def test_dist_worked_examples(ex):
    np.testing.assert_allclose(O.dist(ex["s"], ex["k"]), ex["expect"], rtol=0, atol=1e-15)


@pytest.mark.parametrize("ex", GOLDEN["triple"], ids=lambda e: e["id"])
def test_triple_product_worked_examples(ex):
    np.testing.assert_allclose(O.triple_product_dense(ex["x"], ex["y"], ex["T"]), ex["expect"], atol=1e-15)
    np.testing.assert_allclose(O.triple_product_dp(ex["x"], ex["y"], ex["T"]), ex["expect"], atol=1e-15)


@pytest.mark.parametrize("ex", GOLDEN["const_term"], ids=lambda e: e["id"])
def test_const_term_worked_examples(ex):
    c, c2 = O.const_term(ex["x"], ex["y"], ex["p"], ex["q"])
    np.testing.assert_allclose(2 * (c[:, None] + c2[None, :]), ex["expect_C1"], atol=1e-15)


@pytest.mark.parametrize("ex", GOLDEN["objective"], ids=lambda e: e["id"])
def test_objective_worked_examples(ex):
    assert O.objective(ex["x"], ex["y"], ex["T"]) == pytest.approx(ex["expect"], abs=1e-15)
    assert O.objective_bruteforce(ex["x"], ex["y"], ex["T"]) == pytest.approx(ex["expect"], abs=1e-15)


@pytest.mark.parametrize("ex", GOLDEN["entropy"], ids=lambda e: e["id"])
def test_entropy_worked_examples(ex):
    assert O.entropy(ex["T"]) == pytest.approx(ex["expect"], abs=1e-14)


def test_sinkhorn_worked_example():
    ex = GOLDEN["sinkhorn"][0]
    G = np.array(ex["G"], float)
    f, g, _ = O.sinkhorn(G, np.array(ex["p"]), np.array(ex["q"]), ex["eps"], 200)
    T = O.plan_from_duals(G, f, g, ex["eps"])
    np.testing.assert_allclose(T, ex["expect"], atol=ex["atol"])
    # the closed form itself: sigma = 1/(1+e^{-1/eps})
    sig = 1.0 / (1.0 + math.exp(-1.0 / ex["eps"]))
    np.testing.assert_allclose(T, [[sig / 2, (1 - sig) / 2], [(1 - sig) / 2, sig / 2]], atol=1e-12)


# --------------------------------------------------------------------------- DP vs dense

@pytest.mark.parametrize("n", [1, 2, 3, 7, 64])
@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_dp_distance_matches_dense(n, k):
    """the recursion equals the dense product (<= 1e-12 rel)."""
    rng = np.random.default_rng(n * 10 + k)
    s = _sorted(rng, n)
    if n >= 7:
        s[3] = s[2]  # a tie: zero gap (reading R15)
    v = rng.random(n)
    dense = O.dist(s, k) @ v
    dp = O.ref_dp_distance(v, s, k)
    assert np.max(np.abs(dp - dense)) <= 1e-12 * max(1.0, np.max(np.abs(dense)))
    lower = np.array([sum((s[i] - s[j]) ** k * v[j] for j in range(i)) for i in range(n)])
    np.testing.assert_allclose(O.ref_dp_lower(v, s, k), lower, rtol=1e-12, atol=1e-15)


def test_dp_integer_grid_is_paper_recursion():
    """On the integer grid (h = 1) the gap recursion is the paper's
    a_{i+1,r} = x_i + sum_s C(r-1,s-1) a_{is}: check against a
    direct transcription of that integer formula."""
    n, k = 9, 3
    v = np.random.default_rng(1).random(n)
    a = np.zeros((n, k + 1))
    for i in range(n - 1):
        for r in range(1, k + 2):
            a[i + 1, r - 1] = v[i] + sum(math.comb(r - 1, s - 1) * a[i, s - 1] for s in range(1, r + 1))
    np.testing.assert_allclose(O.ref_dp_lower(v, np.arange(n, dtype=float), k), a[:, k], rtol=1e-14)


def test_triple_product_dp_matches_dense():
    """Paper's exactness claim in fp64: <= 1e-12."""
    rng = np.random.default_rng(3)
    for (n, m, k) in [(12, 9, 1), (40, 33, 1), (17, 23, 2), (21, 14, 3), (9, 16, 5)]:
        x, y = _sorted(rng, n), _sorted(rng, m)
        T = rng.random((n, m))
        dense = O.triple_product_dense(x, y, T, k)
        dp = O.triple_product_dp(x, y, T, k)
        assert np.linalg.norm(dp - dense) <= 1e-12 * np.linalg.norm(dense)


# --------------------------------------------------------------------------- gradient

def test_gradient_three_ways_any_plan():
    """c2 == c4 for any T: entrywise definition vs decomposition."""
    rng = np.random.default_rng(4)
    for (n, m) in [(1, 1), (1, 5), (5, 1), (7, 5), (12, 12)]:
        x, y = _sorted(rng, n), _sorted(rng, m)
        T = rng.random((n, m))
        ge = O.grad_entrywise(x, y, T)
        gr = O.grad_realized(x, y, T)
        assert np.max(np.abs(ge - gr)) <= 1e-12 * max(1.0, np.max(np.abs(ge)))


def test_gradient_prescribed_on_feasible_plan():
    """c3 == c2 iff T in S(p, q) (reading R4); and differs for an infeasible T."""
    rng = np.random.default_rng(5)
    n, m = 8, 6
    x, y = _sorted(rng, n), _sorted(rng, m)
    p, q = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
    T = _feasible_plan(rng, p, q)
    ge = O.grad_entrywise(x, y, T)
    np.testing.assert_allclose(O.grad_prescribed(x, y, p, q, T), ge, atol=1e-12)
    np.testing.assert_allclose(O.grad_prescribed_dp(x, y, p, q, T), ge, atol=1e-12)
    T2 = T * 1.1
    assert np.max(np.abs(O.grad_prescribed(x, y, p, q, T2) - O.grad_entrywise(x, y, T2))) > 1e-3


def test_homogeneity_identity():
    """<grad E(T), T> = 2 E(T) for every T: catches a wrong factor."""
    rng = np.random.default_rng(6)
    x, y = _sorted(rng, 9), _sorted(rng, 7)
    T = rng.random((9, 7))
    eb = O.objective_bruteforce(x, y, T)
    assert np.sum(O.grad_realized(x, y, T) * T) == pytest.approx(2 * eb, rel=1e-12)
    assert O.objective(x, y, T) == pytest.approx(eb, rel=1e-12)


def test_finite_differences():
    """Central differences of the brute-force E match the gradient."""
    rng = np.random.default_rng(7)
    n = 8
    x, y = _sorted(rng, n), _sorted(rng, n)
    T = rng.random((n, n)) / n ** 2
    G = O.grad_realized(x, y, T)
    d = 1e-6
    for (i, p) in [(0, 0), (3, 5), (7, 2), (4, 4)]:
        Tp, Tm = T.copy(), T.copy()
        Tp[i, p] += d
        Tm[i, p] -= d
        fd = (O.objective_bruteforce(x, y, Tp) - O.objective_bruteforce(x, y, Tm)) / (2 * d)
        assert fd == pytest.approx(G[i, p], rel=1e-5)


def test_closed_form_E_of_product_plan():
    """E(p (x) p) on the uniform grid, X = Y, uniform p:
    (N+1)/(3(N-1)) - 2((N+1)/(3N))^2, from E[d^2] = 2 Var and E[d] = (N+1)/(3N)
    of the discrete uniform law (derived from PAPER.md:86)."""
    printed = {2: 0.5, 3: 0.2716049383, 10: 0.1385185185, 256: 0.1119859882}
    for n, val in printed.items():
        x = np.arange(n) / (n - 1)
        p = np.full(n, 1.0 / n)
        closed = (n + 1) / (3 * (n - 1)) - 2 * ((n + 1) / (3 * n)) ** 2
        assert closed == pytest.approx(val, abs=1e-10)
        assert O.objective(x, x, np.outer(p, p)) == pytest.approx(closed, rel=1e-12)


def test_closed_form_first_gradient():
    """G0 = 2(c_i + c'_p) - 4 (D_X p)_i (D_Y q)_p at T0 = p (x) q,
    with the integer-index closed forms on a uniform grid and uniform p."""
    for n in [2, 5, 13]:
        x = np.arange(n) / (n - 1)
        p = np.full(n, 1.0 / n)
        i = np.arange(1, n + 1, dtype=float)
        DXp = ((i - 1) * i / 2 + (n - i) * (n - i + 1) / 2) / (n * (n - 1))
        c = ((i - 1) * i * (2 * i - 1) + (n - i) * (n - i + 1) * (2 * n - 2 * i + 1)) / (6 * n * (n - 1) ** 2)
        G0 = 2 * (c[:, None] + c[None, :]) - 4 * DXp[:, None] * DXp[None, :]
        np.testing.assert_allclose(O.grad_prescribed(x, x, p, p, np.outer(p, p)), G0, atol=1e-14)
        np.testing.assert_allclose(O.grad_entrywise(x, x, np.outer(p, p)), G0, atol=1e-14)


def test_permutation_couplings_bruteforce():
    """N <= 6, uniform weights: E(P_sigma) >= 0; E = 0 at the identity when y = x and
    at the reversal when y = -x (isometries)."""
    rng = np.random.default_rng(8)
    for n in [2, 3, 5, 6]:
        x = _sorted(rng, n)
        best = np.inf
        for sig in itertools.permutations(range(n)):
            P = np.zeros((n, n))
            P[np.arange(n), sig] = 1.0 / n
            e = O.objective(x, x, P)
            assert e >= -1e-15
            best = min(best, e)
        P = np.eye(n) / n
        assert O.objective(x, x, P) == pytest.approx(0.0, abs=1e-15)
        assert best == pytest.approx(0.0, abs=1e-15)
        yr = np.sort(-x)
        R = np.fliplr(np.eye(n)) / n
        assert O.objective(x, yr, R) == pytest.approx(0.0, abs=1e-14)


def test_translation_and_reflection_invariance():
    """GW is invariant to translation / reflection."""
    rng = np.random.default_rng(9)
    n, m = 10, 8
    x, y = _sorted(rng, n), _sorted(rng, m)
    p, q = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
    T = _feasible_plan(rng, p, q)
    G = O.grad_prescribed(x, y, p, q, T)
    np.testing.assert_allclose(O.grad_prescribed(x + 3.7, y - 1.25, p, q, T), G, atol=1e-12)
    # reflection x -> -x reverses the row order (and p); T -> R T
    xr = -x[::-1]
    np.testing.assert_allclose(O.grad_prescribed(xr, y, p[::-1], q, T[::-1]), G[::-1], atol=1e-12)
    assert O.objective(xr, y, T[::-1]) == pytest.approx(O.objective(x, y, T), rel=1e-12)


# --------------------------------------------------------------------------- Sinkhorn

def test_sinkhorn_zero_and_separable_cost():
    """Zero cost -> p (x) q; separable cost a_i + b_p -> p (x) q."""
    rng = np.random.default_rng(10)
    n, m = 6, 4
    p, q = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
    for G in [np.zeros((n, m)), rng.random(n)[:, None] + rng.random(m)[None, :]]:
        f, g, _ = O.sinkhorn(G, p, q, 0.3, 5)
        np.testing.assert_allclose(O.plan_from_duals(G, f, g, 0.3), np.outer(p, q), atol=1e-15)


def test_sinkhorn_marginals_after_each_half_step():
    """After the g-update the column sums are exact; after an f-update the row sums
    are (the two half-steps of PAPER.md:114's Sinkhorn, reading R7)."""
    rng = np.random.default_rng(11)
    G = rng.random((7, 5))
    p, q = rng.dirichlet(np.ones(7)), rng.dirichlet(np.ones(5))
    eps = 0.05
    f, g, _ = O.sinkhorn(G, p, q, eps, 3)
    T = O.plan_from_duals(G, f, g, eps)
    np.testing.assert_allclose(T.sum(0), q, atol=1e-15)
    # one more f half-step from (f, g): rows exact
    f2 = eps * np.log(p) - eps * O.logsumexp((g[None, :] - G) / eps, axis=1)
    np.testing.assert_allclose(O.plan_from_duals(G, f2, g, eps).sum(1), p, atol=1e-15)


def test_sinkhorn_fixed_point_matches_independent_dual_solver():
    """The Sinkhorn limit equals the maximiser of the entropic-OT dual
    max_{f,g} <f,p> + <g,q> - eps sum exp((f_i + g_p - G_ip)/eps), found with
    scipy's L-BFGS (an independent algorithm)."""
    from scipy.optimize import minimize
    rng = np.random.default_rng(12)
    n, m, eps = 4, 3, 0.2
    G = rng.random((n, m))
    p, q = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))

    def negdual(z):
        f, g = z[:n], z[n:]
        K = np.exp((f[:, None] + g[None, :] - G) / eps)
        val = f @ p + g @ q - eps * K.sum()
        grad = np.concatenate([p - K.sum(1), q - K.sum(0)])
        return -val, -grad

    res = minimize(negdual, np.zeros(n + m), jac=True, method="L-BFGS-B",
                   options={"gtol": 1e-14, "ftol": 1e-16, "maxiter": 10000})
    Tref = np.exp((res.x[:n, None] + res.x[None, n:] - G) / eps)
    f, g, _ = O.sinkhorn(G, p, q, eps, 3000)
    np.testing.assert_allclose(O.plan_from_duals(G, f, g, eps), Tref, atol=1e-8)


def test_sinkhorn_tolerance_rule_stops_on_check():
    rng = np.random.default_rng(13)
    G = rng.random((20, 15))
    p, q = rng.dirichlet(np.ones(20)), rng.dirichlet(np.ones(15))
    f, g, used = O.sinkhorn(G, p, q, 0.1, 2000, tol=1e-9, check_every=10)
    assert used % 10 == 0 and used < 2000
    assert O.violation(O.plan_from_duals(G, f, g, 0.1), p, q) <= 1e-9


# --------------------------------------------------------------------------- entropic GW

def test_entropic_gw_single_point():
    """N = M = 1: G = [[0]], T = [[1]], E = 0."""
    r = O.entropic_gw([0.3], [0.7], [1.0], [1.0], 0.01, 3, 10, record_grads=True)
    assert r["T"].tolist() == [[1.0]]
    assert r["gw_objective"] == 0.0
    assert r["G"][0].tolist() == [[0.0]]


def test_entropic_gw_single_row():
    """N = 1 < M: T = q as a row and G = 2 c' exactly (P16b)."""
    rng = np.random.default_rng(14)
    y = _sorted(rng, 6)
    q = rng.dirichlet(np.ones(6))
    r = O.entropic_gw([0.5], y, [1.0], q, 0.01, 2, 20, record_grads=True)
    np.testing.assert_allclose(r["T"][0], q, atol=1e-15)
    c2 = (O.dist(y) ** 2) @ q
    np.testing.assert_allclose(r["G"][1][0], 2 * c2, atol=1e-14)


def test_entropic_gw_large_eps_is_product_plan():
    """eps -> infinity: the entropy term dominates and T -> p (x) q."""
    P = W.uniform_problem(12, 9, seed=1)
    r = O.entropic_gw(P.x, P.y, P.p, P.q, 1e6, 3, 20)
    np.testing.assert_allclose(r["T"], np.outer(P.p, P.q), atol=1e-9)


def test_entropic_gw_reversal_equivariance():
    """Reversing the source (x -> -x reversed, p reversed) gives R T."""
    P = W.uniform_problem(15, 11, seed=2, eps=0.02)
    r1 = O.entropic_gw(P.x, P.y, P.p, P.q, P.eps, 4, 50)
    r2 = O.entropic_gw(-P.x[::-1], P.y, P.p[::-1], P.q, P.eps, 4, 50)
    np.testing.assert_allclose(r2["T"], r1["T"][::-1], atol=1e-12)


def test_entropic_gw_dp_equals_dense_paper_table2():
    """The paper's central exactness claim (||P_FGC - P||_F =
    5.12e-15 at N = 500): on its Table 2 workload (uniform grid, U[0,1] weights,
    k = 1, eps = 0.002, 10 outer iterations), the DP-gradient and dense-gradient
    solves give plans within 1e-12."""
    ex = GOLDEN["paper_table2"][0]
    P = W.table2(ex["N"], seed=0)
    rd = O.entropic_gw(P.x, P.y, P.p, P.q, P.eps, 10, 30, grad_mode="dense")
    rp = O.entropic_gw(P.x, P.y, P.p, P.q, P.eps, 10, 30, grad_mode="dp")
    diff = np.linalg.norm(rd["T"] - rp["T"])
    assert diff <= ex["bound_used"]


def test_entropic_gw_objective_decreases_c1_recipe():
    """C1 recipe (reduced outer count): E(T^l) falls from E(p (x) q) and the plan is
    feasible to Sinkhorn precision."""
    P = W.config1()
    r = O.entropic_gw(P.x, P.y, P.p, P.q, P.eps, 5, 100)
    e0 = O.objective(P.x, P.y, np.outer(P.p, P.q))
    assert r["E"][-1] < r["E"][0] < e0
    assert r["viol"][-1] < 1e-6


# --------------------------------------------------------------------------- FGW

def test_fgw_endpoints():
    """alpha = 1 is GW; alpha = 0 gives Sinkhorn(C o C) after one outer iteration and
    a fixed point afterwards."""
    rng = np.random.default_rng(15)
    n, m = 9, 7
    x, y = _sorted(rng, n), _sorted(rng, m)
    p, q = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
    fx, fy = rng.standard_normal(n), rng.standard_normal(m)
    r1 = O.entropic_fgw(x, y, p, q, fx, fy, 1.0, 0.05, 3, 40)
    rg = O.entropic_gw(x, y, p, q, 0.05, 3, 40)
    np.testing.assert_array_equal(r1["T"], rg["T"])
    r0 = O.entropic_fgw(x, y, p, q, fx, fy, 0.0, 0.05, 3, 40)
    CC = (fx[:, None] - fy[None, :]) ** 2
    f, g, _ = O.sinkhorn(CC, p, q, 0.05, 120)
    np.testing.assert_allclose(r0["T"], O.plan_from_duals(CC, f, g, 0.05), atol=1e-12)


def test_fgw_gradient_bruteforce():
    """grad E_bar = (1-theta) c^2 + theta * 2 sum (d - d)^2 T  on a feasible plan."""
    rng = np.random.default_rng(16)
    n, m, th = 6, 5, 0.3
    x, y = _sorted(rng, n), _sorted(rng, m)
    p, q = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
    fx, fy = rng.standard_normal(n), rng.standard_normal(m)
    T = _feasible_plan(rng, p, q)
    brute = (1 - th) * (fx[:, None] - fy[None, :]) ** 2 + th * O.grad_entrywise(x, y, T)
    np.testing.assert_allclose(O.fgw_grad_prescribed(x, y, p, q, fx, fy, th, T), brute, atol=1e-12)


def test_fgw_objective_closed_form_product_plan():
    """E_bar(p (x) p) = (1 - theta) <C o C, p (x) p> + theta E(p (x) p) with both
    parts in closed form: <(fx - fy)^2, p (x) q> = E_p[fx^2] - 2 E_p[fx] E_q[fy] + E_q[fy^2] (moments of
    the product law) and E(p (x) p) on the uniform grid from P6.  Dropping the (1 - theta) factor, or
    weighting the GW part by anything but theta, fails at theta in (0, 1)."""
    rng = np.random.default_rng(41)
    for n in [2, 7, 30]:
        x = np.arange(n) / (n - 1)
        p = np.full(n, 1.0 / n)
        fx, fy = rng.standard_normal(n), rng.standard_normal(n)
        cc = p @ fx ** 2 - 2 * (p @ fx) * (p @ fy) + p @ fy ** 2
        e_gw = (n + 1) / (3 * (n - 1)) - 2 * ((n + 1) / (3 * n)) ** 2
        for th in [0.0, 0.25, 0.5, 1.0]:
            closed = (1 - th) * cc + th * e_gw
            assert O.fgw_objective(x, x, fx, fy, th, np.outer(p, p)) == pytest.approx(closed, rel=1e-12, abs=1e-15)


def test_fgw_objective_bruteforce_any_plan():
    """E_bar(T) = (1 - theta) sum_ip (fx_i - fy_p)^2 T_ip + theta sum_ijpq (d_ij - d'_pq)^2 T_ip T_jq
    by explicit loops over the entries on a non-feasible random plan."""
    rng = np.random.default_rng(42)
    n, m = 4, 3
    x, y = _sorted(rng, n), _sorted(rng, m)
    fx, fy = rng.standard_normal(n), rng.standard_normal(m)
    T = rng.random((n, m))
    lin = sum((fx[i] - fy[j]) ** 2 * T[i, j] for i in range(n) for j in range(m))
    quad = sum((abs(x[i] - x[j]) - abs(y[a] - y[b])) ** 2 * T[i, a] * T[j, b]
               for i in range(n) for j in range(n) for a in range(m) for b in range(m))
    for th in [0.0, 0.4, 1.0]:
        assert O.fgw_objective(x, y, fx, fy, th, T) == pytest.approx((1 - th) * lin + th * quad, rel=1e-12)


def test_violation_is_two_sided():
    """violation = max(||T1 - p||_inf, ||T^T 1 - q||_inf): on product plans the
    marginals are known in closed form -- p' (x) q has row sums p' and column sums q exactly, p (x) q'
    the reverse -- so a rows-only or columns-only check fails one of the two cases."""
    rng = np.random.default_rng(43)
    n, m = 9, 6
    p, q = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
    p2, q2 = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
    assert O.violation(np.outer(p, q), p, q) == pytest.approx(0.0, abs=1e-16)
    assert O.violation(np.outer(p2, q), p, q) == pytest.approx(np.max(np.abs(p2 - p)), abs=1e-16)
    assert O.violation(np.outer(p, q2), p, q) == pytest.approx(np.max(np.abs(q2 - q)), abs=1e-16)
    # a plan with exact row sums and one column off by d: the violation is d (loop sums)
    T = np.outer(p, q)
    d = 1e-3
    T[0, 0] += d
    T[0, 1] -= d
    rows = max(abs(sum(T[i, :]) - p[i]) for i in range(n))
    cols = max(abs(sum(T[:, j]) - q[j]) for j in range(m))
    assert rows < 1e-15 and cols == pytest.approx(d, rel=1e-9)
    assert O.violation(T, p, q) == pytest.approx(d, rel=1e-9)


# --------------------------------------------------------------------------- streamed (C4-size) evaluations

def _blocks(T, b):
    return [(j, T[j:j + b]) for j in range(0, T.shape[0], b)]


def test_streamed_gradient_rows_cols_match_dense():
    """grad_rows_cols (row blocks of T, D generated blockwise, the paper's recursion for the 1-D
    products) equals the dense definition c3 on the sampled lines, ragged blocks, any plan."""
    rng = np.random.default_rng(51)
    n, m = 157, 131
    x, y = _sorted(rng, n), _sorted(rng, m)
    p, q = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
    T = rng.random((n, m)) / (n * m)
    I = np.sort(rng.choice(n, 9, replace=False))
    J = np.sort(rng.choice(m, 7, replace=False))
    GI, GJ = O.grad_rows_cols(x, y, p, q, _blocks(T, 40), I, J)
    Gd = O.grad_prescribed(x, y, p, q, T)
    np.testing.assert_allclose(GI, Gd[I], rtol=0, atol=1e-13)
    np.testing.assert_allclose(GJ, Gd[:, J], rtol=0, atol=1e-13)
    c, c2 = O.const_term_blocked(x, y, p, q, block=33)
    cd, c2d = O.const_term(x, y, p, q)
    np.testing.assert_allclose(c, cd, rtol=1e-14)
    np.testing.assert_allclose(c2, c2d, rtol=1e-14)


def test_prefix_sum_distance_apply_matches_dense_and_recursion():
    """D v by prefix sums (k = 1) equals the dense product and the paper's recursion
    (PAPER.md:219-243), along either axis, with ties in the support."""
    rng = np.random.default_rng(52)
    s = np.sort(np.concatenate([rng.random(40), [0.5, 0.5, 0.5]]))
    V = rng.random((7, s.size))
    D = O.dist(s)
    np.testing.assert_allclose(O.dist_apply_prefix(V, s, axis=1), V @ D, rtol=0, atol=1e-13)
    np.testing.assert_allclose(O.dist_apply_prefix(V.T, s, axis=0), D @ V.T, rtol=0, atol=1e-13)
    np.testing.assert_allclose(O.dist_apply_prefix(V, s, axis=1), O.ref_dp_distance(V, s), rtol=0, atol=1e-13)


def test_streamed_objective_and_violation_match_dense():
    """objective_k1 (two streamed passes) equals the dense objective and the
    brute-force quadruple sum; violation_streamed equals the dense two-sided violation."""
    rng = np.random.default_rng(53)
    n, m = 211, 97
    x, y = _sorted(rng, n), _sorted(rng, m)
    p, q = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
    T = rng.random((n, m)) / (n * m)
    E = O.objective_k1(x, y, _blocks(T, 50))
    assert O.objective_k1(x, y, _blocks(T, 17), workers=4) == pytest.approx(E, rel=1e-13)
    assert E == pytest.approx(O.objective(x, y, T), rel=1e-12)
    Ts = T[:9, :8] / T[:9, :8].sum()
    assert O.objective_k1(x[:9], y[:8], _blocks(Ts, 4)) == pytest.approx(
        O.objective_bruteforce(x[:9], y[:8], Ts), rel=1e-12)
    assert O.violation_streamed(_blocks(T, 64), p, q) == pytest.approx(O.violation(T, p, q), rel=1e-14)
    # the closed form P6 of E(p (x) p) on the uniform grid
    nn = 300
    g = np.arange(nn) / (nn - 1)
    pp = np.full(nn, 1.0 / nn)
    closed = (nn + 1) / (3 * (nn - 1)) - 2 * ((nn + 1) / (3 * nn)) ** 2
    assert O.objective_k1(g, g, _blocks(np.outer(pp, pp), 64)) == pytest.approx(closed, rel=1e-12)


def test_streamed_fgw_and_ugw_match_dense():
    """C5-size evaluations: fgw_rows_cols / fgw_objective_k1 equal the dense FGW gradient (itself pinned
    by brute force) and objective; ugw_functional_k1 equals the BRUTE-FORCE functional with every
    tensor product formed (tiny) and the dense closed form (larger), zero entries and masses != 1
    included."""
    rng = np.random.default_rng(57)
    n, m = 83, 61
    x, y = _sorted(rng, n), _sorted(rng, m)
    p, q = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
    fx, fy = rng.standard_normal(n), rng.standard_normal(m)
    T = rng.random((n, m)) / (n * m)
    T[rng.random((n, m)) < 0.1] = 0.0
    I, J = np.array([0, 5, 40, n - 1]), np.array([1, 2, 33, m - 1])
    for alpha in (0.0, 0.3, 1.0):
        G = O.fgw_grad_prescribed(x, y, p, q, fx, fy, alpha, T)
        GI, GJ = O.fgw_rows_cols(x, y, p, q, fx, fy, alpha, _blocks(T, 20), I, J)
        np.testing.assert_allclose(GI, G[I], atol=1e-13)
        np.testing.assert_allclose(GJ, G[:, J], atol=1e-13)
        assert O.fgw_objective_k1(x, y, fx, fy, alpha, _blocks(T, 20), workers=2) == pytest.approx(
            O.fgw_objective(x, y, fx, fy, alpha, T), rel=1e-12)
    u, v = 0.7 * p, 1.4 * q
    F, E, mass = O.ugw_functional_k1(x, y, u, v, _blocks(T, 20), 0.8, 0.05)
    assert F == pytest.approx(O.ugw_functional(x, y, u, v, T, 0.8, 0.05), rel=1e-12)
    assert E == pytest.approx(O.objective(x, y, T), rel=1e-12) and mass == pytest.approx(T.sum(), rel=1e-14)
    Ts = T[:5, :4] * 300
    Fs, _, _ = O.ugw_functional_k1(x[:5], y[:4], u[:5], v[:4], _blocks(Ts, 2), 0.8, 0.05)
    assert Fs == pytest.approx(O.ugw_functional_bruteforce(x[:5], y[:4], u[:5], v[:4], Ts, 0.8, 0.05), rel=1e-11)


# --------------------------------------------------------------------------- workloads

def test_workloads_deterministic_and_valid():
    a, b = W.config1(), W.config1()
    np.testing.assert_array_equal(a.x, b.x)
    for P in [W.config1(), W.config2(512), W.config4(1024), W.config5(300, 200), W.table2(50)]:
        assert np.all(np.diff(P.x) >= 0) and np.all(np.diff(P.y) >= 0)
        assert abs(P.p.sum() - 1) < 1e-12 and abs(P.q.sum() - 1) < 1e-12
        assert np.all(P.p >= 0) and np.all(P.q >= 0)
    P3 = W.config3(64)
    T = P3.extra["T"]
    assert T.dtype == np.float32 and np.all(T > 0)
    np.testing.assert_allclose(T.sum(0), P3.q, rtol=1e-5)


# --------------------------------------------------------------------------- 2-D grids (f3)

@pytest.mark.parametrize("ex", GOLDEN["grid2d"], ids=lambda e: e["id"])
def test_grid2d_worked_examples(ex):
    np.testing.assert_allclose(O.apply_distance_2d(ex["v"], ex["axis"], ex["k"]), ex["expect"], atol=1e-15)
    np.testing.assert_allclose(O.dist2d(ex["axis"], ex["k"]) @ np.asarray(ex["v"], float), ex["expect"], atol=1e-15)


def test_dist2d_is_kronecker_sum_at_k1():
    """k = 1: D-hat = D1 (x) J + J (x) D1 (PAPER.md:348 with k = 1), built with np.kron independently."""
    rng = np.random.default_rng(0)
    s = np.sort(rng.random(6))
    D1 = np.abs(s[:, None] - s[None, :])
    J = np.ones((6, 6))
    np.testing.assert_allclose(O.dist2d(s, 1), np.kron(D1, J) + np.kron(J, D1), atol=1e-15)
    # uniform grid: h (|a - a'| + |b - b'|)
    h = 0.25
    g = h * np.arange(5)
    idx = np.array([(a, b) for a in range(5) for b in range(5)])
    man = np.abs(idx[:, None, 0] - idx[None, :, 0]) + np.abs(idx[:, None, 1] - idx[None, :, 1])
    np.testing.assert_allclose(O.dist2d(g, 2), (h * man) ** 2, atol=1e-14)


@pytest.mark.parametrize("k", [1, 2, 3])
def test_apply_distance_2d_matches_dense(k):
    rng = np.random.default_rng(k)
    s = np.sort(rng.random(9))
    v = rng.random(81)
    np.testing.assert_allclose(O.apply_distance_2d(v, s, k), O.dist2d(s, k) @ v, rtol=1e-12)


def test_grad_2d_bruteforce_and_objective():
    """2-D gradient: against the entrywise definition 2 sum_{jq} (d_ij - d_pq)^2 T_jq
     on a feasible plan, brute force; <G, T> = 2E (P8)."""
    rng = np.random.default_rng(4)
    sx, sy = np.sort(rng.random(3)), np.sort(rng.random(2))
    N, M = 9, 4
    p, q = rng.dirichlet(np.ones(N)), rng.dirichlet(np.ones(M))
    T = _feasible_plan(rng, p, q)
    DX, DY = O.dist2d(sx), O.dist2d(sy)
    Gb = np.zeros((N, M))
    for i in range(N):
        for pp in range(M):
            Gb[i, pp] = 2.0 * np.sum((DX[i][:, None] - DY[pp][None, :]) ** 2 * T)
    G = O.grad_prescribed_2d(sx, sy, p, q, T)
    np.testing.assert_allclose(G, Gb, rtol=1e-12, atol=1e-13)
    E = O.objective_2d(sx, sy, T)
    Eb = sum(((DX[i, j] - DY[a, b]) ** 2) * T[i, a] * T[j, b]
             for i in range(N) for j in range(N) for a in range(M) for b in range(M))
    assert abs(E - Eb) <= 1e-12 * max(1.0, abs(Eb))
    assert abs(np.sum(G * T) - 2.0 * E) <= 1e-12


def test_entropic_gw_2d_grid_reflection_equivariance():
    """Reflecting one axis of the x grid (a -> n-1-a, with the marginal permuted alike) leaves the
    objective trajectory unchanged (GW is invariant under isometries)."""
    rng = np.random.default_rng(9)
    n = 4
    s = np.arange(n) / (n - 1.0)
    p, q = rng.dirichlet(np.ones(n * n)), rng.dirichlet(np.ones(n * n))
    r1 = O.entropic_gw_2d(s, s, p, q, 0.05, 3, 40)
    perm = np.array([(n - 1 - a) * n + b for a in range(n) for b in range(n)])
    r2 = O.entropic_gw_2d(s, s, p[perm], q, 0.05, 3, 40)
    np.testing.assert_allclose(r1["E"], r2["E"], rtol=1e-9)


def test_fgw_2d_bruteforce_and_reductions():
    """FGW on 2-D grids (Remark 2): the gradient against the entrywise
    (1 - a) c_ip^2 + a * 2 sum_{jq} (d_ij - d_pq)^2 T_jq on a feasible plan; alpha = 1 is GW."""
    rng = np.random.default_rng(14)
    sx, sy = np.sort(rng.random(3)), np.sort(rng.random(3))
    N, M = 9, 9
    p, q = rng.dirichlet(np.ones(N)), rng.dirichlet(np.ones(M))
    fx, fy = rng.random(N), rng.random(M)
    T = _feasible_plan(rng, p, q)
    DX, DY = O.dist2d(sx), O.dist2d(sy)
    a = 0.3
    Gb = np.zeros((N, M))
    for i in range(N):
        for pp in range(M):
            Gb[i, pp] = (1 - a) * (fx[i] - fy[pp]) ** 2 + a * 2.0 * np.sum((DX[i][:, None] - DY[pp][None, :]) ** 2 * T)
    np.testing.assert_allclose(O.fgw_grad_prescribed_2d(sx, sy, p, q, fx, fy, a, T), Gb, rtol=1e-12, atol=1e-13)
    Eb = sum((1 - a) * (fx[i] - fy[pp]) ** 2 * T[i, pp] for i in range(N) for pp in range(M)) + a * sum(
        ((DX[i, j] - DY[u, v]) ** 2) * T[i, u] * T[j, v]
        for i in range(N) for j in range(N) for u in range(M) for v in range(M))
    assert abs(O.fgw_objective_2d(sx, sy, fx, fy, a, T) - Eb) <= 1e-12
    r1 = O.entropic_fgw_2d(sx, sy, p, q, fx, fy, 1.0, 0.05, 2, 30)
    r2 = O.entropic_gw_2d(sx, sy, p, q, 0.05, 2, 30)
    np.testing.assert_allclose(r1["E"], r2["E"], rtol=1e-12)


def test_mirror_descent_general_tau_is_the_kl_proximal_step():
    """with tau != eps the oracle's step solves the cost Pi = G + (eps - tau) ln T^l at
    regulariser tau; that must equal the KL-proximal step argmin <grad E + eps grad H(T^l), T> +
    tau KL(T|T^l) over S(p,q), minimised directly (scipy, tiny instance), at the first TWO steps."""
    rng = np.random.default_rng(21)
    n, m = 3, 4
    x, y = np.sort(rng.random(n)), np.sort(rng.random(m))
    p, q = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
    eps, tau = 0.08, 0.03
    r1 = O.entropic_gw(x, y, p, q, eps, 1, 4000, tau=tau)
    Tl = np.outer(p, q)
    _check_kl_proximal_step(x, y, p, q, eps, tau, Tl, r1["T"])
    # second step: ln T^1 is no longer separable (on T^0 = p (x) q the (eps - tau) ln T^0 term only shifts
    # the duals, so the first step alone cannot see its sign)
    r2 = O.entropic_gw(x, y, p, q, eps, 2, 4000, tau=tau)
    _check_kl_proximal_step(x, y, p, q, eps, tau, r1["T"], r2["T"])
    for t2 in (0.03, 0.2):  # and the sign matters: tau on either side of eps gives different plans
        assert np.max(np.abs(O.entropic_gw(x, y, p, q, eps, 2, 4000, tau=t2)["T"]
                             - O.entropic_gw(x, y, p, q, eps, 2, 4000)["T"])) > 1e-4
    # tau = eps is the default path exactly
    a = O.entropic_gw(x, y, p, q, eps, 3, 50)
    b = O.entropic_gw(x, y, p, q, eps, 3, 50, tau=eps)
    np.testing.assert_array_equal(a["T"], b["T"])


def _check_kl_proximal_step(x, y, p, q, eps, tau, Tl, T_next):
    from scipy.optimize import minimize
    n, m = Tl.shape
    G = O.grad_prescribed(x, y, p, q, Tl)
    C = G + eps * np.log(Tl)  # grad E + eps grad H(T^l)

    # parametrise S(p, q) feasibly: T = T^l + B z with B spanning {sum rows = sum cols = 0}
    basis = []
    for i in range(n - 1):
        for j in range(m - 1):
            Bm = np.zeros((n, m))
            Bm[i, j], Bm[i, m - 1], Bm[n - 1, j], Bm[n - 1, m - 1] = 1, -1, -1, 1
            basis.append(Bm)
    basis = np.array(basis)

    def obj(z):
        T = Tl + np.tensordot(z, basis, 1)
        if np.any(T <= 0):
            return 1e9, np.zeros_like(z)
        val = np.sum(C * T) + tau * np.sum(T * np.log(T / Tl) - T + Tl)
        dT = C + tau * np.log(T / Tl)
        return val, np.tensordot(basis, dT, ([1, 2], [0, 1]))

    r = minimize(obj, np.zeros(len(basis)), jac=True, method="L-BFGS-B",
                 options={"ftol": 1e-15, "gtol": 1e-12, "maxiter": 5000})
    Tp = Tl + np.tensordot(r.x, basis, 1)
    np.testing.assert_allclose(T_next, Tp, atol=1e-8)


# --------------------------------------------------------------------------- result fields / wiring

def test_entropic_objective_field_closed_form_and_duality():
    """The reported entropic objective is E(T) + eps H(T), H = sum T (ln T - 1).
    (i) outer = 0: T = p (x) p uniform on the uniform grid, where E has the closed form P6 and
    H(p (x) p) = -2 ln N - 1.  (ii) after converged inner loops T = exp((f + g - G)/eps) is feasible, so
    eps H(T) = <f, p> + <g, q> - <G, T> - eps (Gibbs form + marginals; no logarithm of T taken here)."""
    n, eps = 10, 0.07
    x = np.arange(n) / (n - 1)
    p = np.full(n, 1.0 / n)
    r0 = O.entropic_gw(x, x, p, p, eps, 0, 5)
    closed = (n + 1) / (3 * (n - 1)) - 2 * ((n + 1) / (3 * n)) ** 2
    assert r0["entropic_objective"] == pytest.approx(closed + eps * (-2 * math.log(n) - 1), rel=1e-12)
    rng = np.random.default_rng(31)
    n, m = 7, 5
    x, y = _sorted(rng, n), _sorted(rng, m)
    p, q = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
    fx, fy = rng.standard_normal(n), rng.standard_normal(m)
    r = O.entropic_gw(x, y, p, q, eps, 3, 3000, record_grads=True)
    G, T = r["G"][-1], r["T"]
    dual = r["f"] @ p + r["g"] @ q - np.sum(G * T) - eps
    assert r["entropic_objective"] - r["gw_objective"] == pytest.approx(dual, rel=1e-9)
    assert r["entropic_objective"] - r["gw_objective"] < 0 < r["gw_objective"]
    # FGW: same identity with the FGW gradient of the previous plan as the cost
    alpha = 0.4
    rf2 = O.entropic_fgw(x, y, p, q, fx, fy, alpha, eps, 2, 3000)
    rf3 = O.entropic_fgw(x, y, p, q, fx, fy, alpha, eps, 3, 3000)
    Gf = O.fgw_grad_prescribed(x, y, p, q, fx, fy, alpha, rf2["T"])
    dual = rf3["f"] @ p + rf3["g"] @ q - np.sum(Gf * rf3["T"]) - eps
    assert rf3["entropic_objective"] - rf3["gw_objective"] == pytest.approx(dual, rel=1e-9)


def test_entropic_fgw_wiring_intermediate_alpha():
    """Remark 2: every FGW outer step is the entropic OT problem of the cost
    grad E_bar(T^l).  With converged inner loops the step's plan is the unique minimiser, so it must
    equal the Sinkhorn fixed point of that cost from a cold start, with the features on the right
    sides (fx on rows, fy on columns: N != M makes a swap an error, equal sizes would hide it, so both)."""
    rng = np.random.default_rng(33)
    for n, m in ((6, 6), (7, 4)):
        x, y = _sorted(rng, n), _sorted(rng, m)
        p, q = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
        fx, fy = rng.standard_normal(n), rng.standard_normal(m)
        alpha, eps = 0.3, 0.08
        T = np.outer(p, q)
        for l in range(1, 3):
            C = np.empty((n, m))
            for i in range(n):
                for j in range(m):
                    C[i, j] = (1 - alpha) * (fx[i] - fy[j]) ** 2
            C += alpha * O.grad_entrywise(x, y, T)  # T in S(p, q): realised = prescribed marginals
            f, g, _ = O.sinkhorn(C, p, q, eps, 4000)
            T = O.plan_from_duals(C, f, g, eps)
            r = O.entropic_fgw(x, y, p, q, fx, fy, alpha, eps, l, 4000)
            np.testing.assert_allclose(r["T"], T, atol=1e-10)
            val = (1 - alpha) * sum((fx[i] - fy[j]) ** 2 * T[i, j] for i in range(n) for j in range(m)) \
                + alpha * O.objective_bruteforce(x, y, T)
            assert r["gw_objective"] == pytest.approx(val, rel=1e-8)


def test_grid_points_flattening():
    """Row i = a n + b of a 2-D grid is the point (axis[a], axis[b]) (reading R31)."""
    P = O.grid_points([0.0, 0.5, 2.0])
    assert P.shape == (9, 2)
    assert tuple(P[1]) == (0.0, 0.5) and tuple(P[3]) == (0.5, 0.0) and tuple(P[5]) == (0.5, 2.0)


def test_entropic_gw_restart_from_T0_is_the_next_step():
    """T0 (reading R5) is the plan the first gradient is evaluated on: with converged inner loops each
    step's plan is the unique minimiser of PAPER.md:108-114, so two steps from p (x) q equal one step
    restarted from the first step's plan (the duals restart from zero; the minimiser does not care)."""
    rng = np.random.default_rng(35)
    n, m = 6, 8
    x, y = _sorted(rng, n), _sorted(rng, m)
    p, q = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
    eps = 0.06
    r1 = O.entropic_gw(x, y, p, q, eps, 1, 4000)
    r2 = O.entropic_gw(x, y, p, q, eps, 2, 4000)
    rr = O.entropic_gw(x, y, p, q, eps, 1, 4000, T0=r1["T"])
    np.testing.assert_allclose(rr["T"], r2["T"], atol=1e-11)
    assert np.max(np.abs(r2["T"] - r1["T"])) > 1e-4
    rf1 = O.entropic_fgw(x, y, p, q, x[::-1], y, 0.5, eps, 1, 4000)
    rf2 = O.entropic_fgw(x, y, p, q, x[::-1], y, 0.5, eps, 2, 4000)
    rfr = O.entropic_fgw(x, y, p, q, x[::-1], y, 0.5, eps, 1, 4000, T0=rf1["T"])
    np.testing.assert_allclose(rfr["T"], rf2["T"], atol=1e-11)
