"""Oracle for entropic unbalanced GW (Remark 3).

Float64 NumPy, test infrastructure only (see oracle/__init__.py).

Remark 3 fixes the functional and the subproblem solved at each iteration
for an updated plan G^:

    min_{G >= 0} < 1/2 grad E(G^) + g(G^), G > + m(G^) (rho KL(G1|u) + rho KL(G^T 1|v) + eps KL(G|u v)),

with m(G^) = 1^T G^ 1, but leaves g(G^) undefined and cites the UGW paper for the rest.  The
readings taken here (R32-R35; the oracle and the GPU take the same ones):

R32  g(G^) is the scalar  rho <log(a/u), a> + rho <log(b/v), b> + eps <log(G^/(u v)), G^>,
     a = G^ 1, b = G^T 1: the part of 1/2 grad F_eps(G^) (F_eps below) that the linearised
     KL penalties do not already carry.  Pinned by finite differences of F_eps
     (tests/test_oracle_pins.py::test_ugw_cost_is_half_gradient_of_functional).
R33  the entropic functional is F_eps(G) = E(G) + rho KL(a (x) a | u (x) u)
     + rho KL(b (x) b | v (x) v) + eps KL(G (x) G | (u v) (x) (u v)) (PAPER.md:150-153 plus the
     entropic term whose linearisation is the subproblem's eps KL(G|u v)); KL(x|y) =
     sum x log(x/y) - m(x) + m(y) (PAPER.md:104 for the plain case).
R34  the subproblem is solved by unbalanced Sinkhorn in log form:
       f = -k eps~ LSE_p((g - C)/eps~ + log v),  g = -k eps~ LSE_i((f - C)/eps~ + log u),
       k = rho~ / (rho~ + eps~),  rho~ = m(G^) rho,  eps~ = m(G^) eps,
     G = exp((f + g - C)/eps~) u v; f-update then g-update (as R7), f = g = 0 before the first
     sweep, warm start across outer iterations.  Pinned by direct minimisation of the
     subproblem's primal on a tiny instance.
R35  G^0 = u v / sqrt(m(u) m(v)), and after each subproblem the plan is rescaled by
     sqrt(m(G^) / m(G)) (mass balance of the UGW iteration).
The rho -> infinity limit is balanced entropic GW at 2 eps with realised-marginal gradients
(pinned against oracle.entropic_gw).  The loop as a whole (R32-R35 together) is pinned by what the
functional fixes: Remark 3 minimises F_eps over all positive measures, so a fixed point of the
iteration must have grad F_eps = 0 entrywise -- checked by central differences of the brute-force
functional with m(u) != m(v) != 1 (tests/test_oracle_ugw.py::
test_ugw_fixed_point_is_a_critical_point_of_the_functional; the mutations "rho~ = rho", "no square
root in R35", "eps for rho in g" all move the fixed point off the critical set,
profiles/r02_oracle_mutations.log).  What stays without a pin is the TRAJECTORY towards that fixed
point (the paper gives no worked example for UGW and several iterations share the fixed point): for
the per-iteration values the reading is still "parity unpinned".
"""

import math

import numpy as np

from .gw import grad_prescribed, objective
from .solver import logsumexp

__all__ = ["kl", "kl_tensor_sq", "ugw_functional", "ugw_functional_bruteforce", "ugw_cost",
           "unbalanced_sinkhorn", "unbalanced_plan", "entropic_ugw"]


def _f64(a):
    return np.asarray(a, dtype=np.float64)


def _xlogy(x, y):
    x, y = _f64(x), _f64(y)
    out = np.zeros(np.broadcast(x, y).shape)
    pos = x > 0
    out[pos] = (x * np.log(np.where(pos, x, 1.0) / np.where(pos, y, 1.0)))[pos]
    return out


def kl(x, y):
    """KL(x|y) = sum x log(x/y) - m(x) + m(y), 0 log 0 = 0 (R33)."""
    x, y = _f64(x), _f64(y)
    return float(np.sum(_xlogy(x, y)) - x.sum() + y.sum())


def kl_tensor_sq(x, y):
    """KL(x (x) x | y (x) y) = 2 m(x) <log(x/y), x> - m(x)^2 + m(y)^2 (closed form of R33's terms)."""
    x, y = _f64(x), _f64(y)
    return float(2.0 * x.sum() * np.sum(_xlogy(x, y)) - x.sum() ** 2 + y.sum() ** 2)


def ugw_functional(x, y, u, v, G, rho, eps, k=1):
    """F_eps(G) (R33): E(G) with realised marginals + the three tensorised KLs."""
    G = _f64(G)
    a, b = G.sum(1), G.sum(0)
    uv = np.outer(_f64(u), _f64(v))
    return (objective(x, y, G, k) + rho * kl_tensor_sq(a, u) + rho * kl_tensor_sq(b, v)
            + eps * kl_tensor_sq(G.ravel(), uv.ravel()))


def ugw_functional_bruteforce(x, y, u, v, G, rho, eps, k=1):
    """F_eps(G) with every tensor product formed explicitly (tiny inputs only)."""
    G = _f64(G)
    x, y, u, v = _f64(x), _f64(y), _f64(u), _f64(v)
    DX = np.abs(x[:, None] - x[None, :]) ** k
    DY = np.abs(y[:, None] - y[None, :]) ** k
    E = np.einsum("ijpq,ip,jq->", (DX[:, :, None, None] - DY[None, None, :, :]) ** 2, G, G)
    a, b = G.sum(1), G.sum(0)
    uv = np.outer(u, v)
    return (E + rho * kl(np.outer(a, a), np.outer(u, u)) + rho * kl(np.outer(b, b), np.outer(v, v))
            + eps * kl(np.outer(G.ravel(), G.ravel()), np.outer(uv.ravel(), uv.ravel())))


def ugw_cost(x, y, u, v, Gh, rho, eps, k=1):
    """C = 1/2 grad E(G^) + g(G^) (reading R32).

    1/2 grad E(G^)_ip = sum_jq (d_ij - d_pq)^2 G^_jq = ((D o D) a)_i + ((D o D) b)_p - 2 (D_X G^ D_Y)_ip
    with the REALISED marginals a, b of G^: G^ is not in S(u, v)."""
    Gh = _f64(Gh)
    a, b = Gh.sum(1), Gh.sum(0)
    half = 0.5 * grad_prescribed(x, y, a, b, Gh, k)
    gsc = (rho * np.sum(_xlogy(a, u)) + rho * np.sum(_xlogy(b, v))
           + eps * np.sum(_xlogy(Gh, np.outer(_f64(u), _f64(v)))))
    return half + gsc


def unbalanced_plan(C, u, v, f, g, eps_t):
    """G = exp((f + g - C)/eps~) u v (R34)."""
    return np.exp((f[:, None] + g[None, :] - _f64(C)) / eps_t) * np.outer(_f64(u), _f64(v))


def unbalanced_sinkhorn(C, u, v, rho_t, eps_t, iters, f0=None, g0=None):
    """`iters` unbalanced Sinkhorn iterations (R34), each an f-update then a g-update."""
    C, u, v = _f64(C), _f64(u), _f64(v)
    with np.errstate(divide="ignore"):
        lu, lv = np.log(u), np.log(v)
    kap = rho_t / (rho_t + eps_t)
    f = np.zeros(C.shape[0]) if f0 is None else _f64(f0).copy()
    g = np.zeros(C.shape[1]) if g0 is None else _f64(g0).copy()
    for _ in range(int(iters)):
        f = -kap * eps_t * logsumexp((g[None, :] - C) / eps_t + lv[None, :], axis=1)
        g = -kap * eps_t * logsumexp((f[:, None] - C) / eps_t + lu[:, None], axis=0)
    return f, g


def entropic_ugw(x, y, u, v, rho, eps, outer, inner, k=1):
    """Entropic UGW iteration (Remark 3 with readings R32-R35).  Returns T, f, g and per outer
    iteration F (= F_eps of the rescaled plan), E (its GW part), mass."""
    u, v = _f64(u), _f64(v)
    G = np.outer(u, v) / math.sqrt(u.sum() * v.sum())
    f = np.zeros(u.size)
    g = np.zeros(v.size)
    out = {"F": [], "E": [], "mass": []}
    for _ in range(int(outer)):
        C = ugw_cost(x, y, u, v, G, rho, eps, k)
        mh = G.sum()
        f, g = unbalanced_sinkhorn(C, u, v, mh * rho, mh * eps, inner, f, g)
        Gn = unbalanced_plan(C, u, v, f, g, mh * eps)
        G = math.sqrt(mh / Gn.sum()) * Gn
        out["F"].append(ugw_functional(x, y, u, v, G, rho, eps, k))
        out["E"].append(objective(x, y, G, k))
        out["mass"].append(float(G.sum()))
    out.update(T=G, f=f, g=g)
    return out
