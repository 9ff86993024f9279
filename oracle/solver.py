"""Oracle: log-domain Sinkhorn and the entropic (F)GW mirror-descent loop.

Float64 NumPy, test infrastructure only (see oracle/__init__.py).

Schedule (reading R7): one Sinkhorn iteration is an f-update
then a g-update; f = g = 0 before the very first sweep of a solve; the duals are
warm-started across outer iterations; the plan is rebuilt from the final (f, g).
The paper states none of this (it only says the subproblem "can be solved with
the Sinkhorn algorithm"), so the schedule is part of the
contract and the GPU path follows it exactly.
"""

import numpy as np

from .gw import grad_prescribed, grad_prescribed_dp, fgw_grad_prescribed, objective, fgw_objective, entropy, violation

__all__ = ["logsumexp", "sinkhorn", "entropic_gw", "entropic_fgw"]


def logsumexp(a, axis):
    """Max-shifted log-sum-exp (a library-style primitive used as one step)."""
    a = np.asarray(a, dtype=np.float64)
    m = np.max(a, axis=axis, keepdims=True)
    m = np.where(np.isfinite(m), m, 0.0)
    s = np.sum(np.exp(a - m), axis=axis, keepdims=True)
    with np.errstate(divide="ignore"):
        out = np.log(s) + m
    return np.squeeze(out, axis=axis)


def _log(v):
    with np.errstate(divide="ignore"):
        return np.log(np.asarray(v, dtype=np.float64))


def plan_from_duals(G, f, g, eps):
    """T_ip = exp((f_i + g_p - G_ip) / eps)  -- the Gibbs form of the entropic-OT
    solution with cost G at regulariser eps (Remark 1)."""
    return np.exp((f[:, None] + g[None, :] - np.asarray(G, np.float64)) / eps)


def sinkhorn(G, p, q, eps, iters, f0=None, g0=None, tol=None, check_every=10):
    """Log-domain Sinkhorn for min <G, T> + eps H(T) over S(p, q).

    PAPER.md:108-114 (eq. "GW sinkhorn": an entropic OT problem with cost Pi,
    "solved with the Sinkhorn algorithm"); with tau = eps, Pi = grad E
    (PAPER.md:128-131).  Each iteration:
        f_i = eps ln p_i - eps LSE_p((g_p - G_ip) / eps)
        g_p = eps ln q_p - eps LSE_i((f_i - G_ip) / eps)
    ``iters`` is the number of (f, g) pairs.  With ``tol`` set, the plan's
    marginal violation is checked after every ``check_every`` iterations and
    the loop stops once it is <= tol (``iters`` is then the cap).
    Returns (f, g, used_iterations).
    """
    G = np.asarray(G, dtype=np.float64)
    n, m = G.shape
    lp, lq = _log(p), _log(q)
    f = np.zeros(n) if f0 is None else np.array(f0, dtype=np.float64)
    g = np.zeros(m) if g0 is None else np.array(g0, dtype=np.float64)
    used = 0
    for it in range(int(iters)):
        f = eps * lp - eps * logsumexp((g[None, :] - G) / eps, axis=1)
        g = eps * lq - eps * logsumexp((f[:, None] - G) / eps, axis=0)
        used = it + 1
        if tol is not None and used % check_every == 0:
            if violation(plan_from_duals(G, f, g, eps), p, q) <= tol:
                break
    return f, g, used


def entropic_gw(x, y, p, q, eps, outer, inner, k=1, T0=None, tol=None,
                check_every=10, record_grads=False, grad_mode="dense", tau=None, cost_dtype=None):
    """Entropic GW by mirror descent with tau = eps.

    PAPER.md:102-114 (eqs. "GW proximal gradient", "GW sinkhorn") and Remark 1
    (PAPER.md:127-133): T^{l} = argmin_{T in S(p,q)} <grad E(T^{l-1}), T> + eps H(T).
    T^0 = p (x) q (reading R5); gradient with the prescribed-
    marginal constant term (reading R4); ``grad_mode="dp"`` evaluates it with the
    paper's recursion instead of dense products.  ``inner`` is an int (same count every
    outer iteration) or a sequence of per-outer counts (to replay the GPU's
    counts under reading R8).

    ``tau`` (default eps): the general mirror-descent step of PAPER.md:102-110,
    T^{l+1} = argmin_{T in S(p,q)} <grad E(T^l) + (eps - tau) grad H(T^l), T> + tau H(T),
    grad H(T) = ln T, i.e. entropic OT of the cost Pi = G + (eps - tau) ln T^l at
    regulariser tau; ln T^l is the log-domain plan (f + g - Pi_prev)/tau (ln p + ln q for
    T^0 = p (x) q), never log of an underflowed entry.

    ``cost_dtype`` (diagnostic only, default None = float64 throughout): round the cost of every
    subproblem to this storage type (e.g. np.float32, the matrix storage BASELINE.json's configs
    prescribe) before the Sinkhorn iterations -- a model of a solver that STORES G in fp32; the
    arithmetic stays float64.  Not the parity contract (the oracle is float64).

    Returns a dict: T, f, g, E (list, E(T^l) for l = 1..L), viol (list),
    inner_used (list), gw_objective, entropic_objective, and G (list) when
    record_grads.
    """
    x = np.asarray(x, np.float64)
    y = np.asarray(y, np.float64)
    p = np.asarray(p, np.float64)
    q = np.asarray(q, np.float64)
    T = np.outer(p, q) if T0 is None else np.array(T0, dtype=np.float64)
    f = np.zeros(x.size)
    g = np.zeros(y.size)
    counts = [int(inner)] * outer if np.isscalar(inner) else [int(c) for c in inner]
    out = {"E": [], "viol": [], "inner_used": [], "G": []}
    tau = eps if tau is None else float(tau)
    if tau != eps:
        lnT = _log(T)  # T^0 (p (x) q or T0); afterwards the log-domain plan
    for l in range(outer):
        if grad_mode == "dp":
            G = grad_prescribed_dp(x, y, p, q, T, k)
        else:
            G = grad_prescribed(x, y, p, q, T, k)
        if tau != eps:
            G = G + (eps - tau) * lnT  # the cost Pi of PAPER.md:110
        if cost_dtype is not None:
            G = G.astype(cost_dtype).astype(np.float64)
        f, g, used = sinkhorn(G, p, q, tau, counts[l], f, g, tol=tol, check_every=check_every)
        T = plan_from_duals(G, f, g, tau)
        if tau != eps:
            lnT = (f[:, None] + g[None, :] - G) / tau
        out["E"].append(objective(x, y, T, k))
        out["viol"].append(violation(T, p, q))
        out["inner_used"].append(used)
        if record_grads:
            out["G"].append(G)
    out.update(T=T, f=f, g=g, gw_objective=out["E"][-1] if outer else objective(x, y, T, k))
    out["entropic_objective"] = out["gw_objective"] + eps * entropy(T)
    return out


def entropic_fgw(x, y, p, q, fx, fy, alpha, eps, outer, inner, k=1, T0=None,
                 tol=None, check_every=10, tau=None):
    """Entropic FGW: the same iteration with grad E_bar (Remark 2, PAPER.md:134-147:
    "The iteration formula ... applies to FGW as well"); ``tau`` as in entropic_gw."""
    x = np.asarray(x, np.float64)
    y = np.asarray(y, np.float64)
    p = np.asarray(p, np.float64)
    q = np.asarray(q, np.float64)
    T = np.outer(p, q) if T0 is None else np.array(T0, dtype=np.float64)
    f = np.zeros(x.size)
    g = np.zeros(y.size)
    counts = [int(inner)] * outer if np.isscalar(inner) else [int(c) for c in inner]
    out = {"E": [], "viol": [], "inner_used": []}
    tau = eps if tau is None else float(tau)
    if tau != eps:
        lnT = _log(T)
    for l in range(outer):
        G = fgw_grad_prescribed(x, y, p, q, fx, fy, alpha, T, k)
        if tau != eps:
            G = G + (eps - tau) * lnT
        f, g, used = sinkhorn(G, p, q, tau, counts[l], f, g, tol=tol, check_every=check_every)
        T = plan_from_duals(G, f, g, tau)
        if tau != eps:
            lnT = (f[:, None] + g[None, :] - G) / tau
        out["E"].append(fgw_objective(x, y, fx, fy, alpha, T, k))
        out["viol"].append(violation(T, p, q))
        out["inner_used"].append(used)
    out.update(T=T, f=f, g=g, gw_objective=out["E"][-1])
    out["entropic_objective"] = out["gw_objective"] + eps * entropy(T)
    return out
