"""Oracle for 2-D grids (the paper's §3.1 / Table 3 workload).

Float64 NumPy, test infrastructure only (see oracle/__init__.py).

Points of an n x n tensor grid with axis coordinates s_0 <= ... <= s_{n-1} are indexed
i = a n + b <-> (s_a, s_b) (reading R31: the paper flattens mat(u) with its vec(), PAPER.md:350-353;
any fixed flattening gives the same GW problem).  The distance is the Manhattan distance raised to
the power k, the paper's D_X = h^k D-hat (whose block matrix is garbled; reading
R31): d_ij = (|s_a - s_a'| + |s_b - s_b'|)^k.  On the uniform grid s_a = a h this is exactly
h^k (|a - a'| + |b - b'|)^k.
"""

import math

import numpy as np

from .gw import entropy, violation
from .solver import sinkhorn, plan_from_duals

__all__ = ["grid_points", "dist2d", "apply_distance_2d", "grad_prescribed_2d", "objective_2d",
           "entropic_gw_2d", "fgw_grad_prescribed_2d", "fgw_objective_2d", "entropic_fgw_2d"]

DENSE_GUARD = 16384


def _f64(a):
    return np.asarray(a, dtype=np.float64)


def grid_points(axis):
    """(n^2, 2) coordinates, row i = a n + b -> (axis[a], axis[b])."""
    s = _f64(axis)
    A, B = np.meshgrid(s, s, indexing="ij")
    return np.stack([A.ravel(), B.ravel()], axis=1)


def dist2d(axis, k=1, force=False):
    """Dense D[i, j] = (|s_a - s_a'| + |s_b - s_b'|)^k (reading R31)."""
    P = grid_points(axis)
    if P.shape[0] > DENSE_GUARD and not force:
        raise ValueError("dist2d: %d points exceed the dense guard" % P.shape[0])
    man = np.abs(P[:, None, 0] - P[None, :, 0]) + np.abs(P[:, None, 1] - P[None, :, 1])
    return man ** k


def apply_distance_2d(v, axis, k=1):
    """D-hat v by the paper's Kronecker expansion (eq. "2D kronecker"):
        D-hat = sum_r C(k, r) D1^{o r} (x) D1^{o (k - r)},
        D-hat v = sum_r C(k, r) vec(D1^{o r} mat(v) D1^{o (k - r)})
    with D1 the 1-D axis distance matrix and mat(v)[a, b] = v[a n + b] (the flattening of
    grid_points).  D1^{o 0} is the all-ones matrix J."""
    s = _f64(axis)
    n = s.size
    D1 = np.abs(s[:, None] - s[None, :])
    V = _f64(v).reshape(n, n)
    out = np.zeros((n, n))
    for r in range(k + 1):
        out += math.comb(k, r) * (D1 ** r) @ V @ (D1 ** (k - r)).T
    return out.ravel()


def grad_prescribed_2d(axis_x, axis_y, p, q, T, k=1):
    """G = 2((D_X o D_X) p 1^T + 1 ((D_Y o D_Y) q)^T) - 4 D_X T D_Y on 2-D grids (the decomposition of
    PAPER.md:120-126 with the 2-D distance of PAPER.md:300-336; the 2-D product is PAPER.md:341-343,
    eq. "2d gradient"), dense."""
    DX, DY = dist2d(axis_x, k), dist2d(axis_y, k)
    T = _f64(T)
    c = (DX * DX) @ _f64(p)
    c2 = (DY * DY) @ _f64(q)
    return 2.0 * (c[:, None] + c2[None, :]) - 4.0 * (DX @ T @ DY)


def objective_2d(axis_x, axis_y, T, k=1):
    """E(T) = a^T (D_X o D_X) a + b^T (D_Y o D_Y) b - 2 <D_X T D_Y, T>, realised marginals."""
    DX, DY = dist2d(axis_x, k), dist2d(axis_y, k)
    T = _f64(T)
    a, b = T.sum(1), T.sum(0)
    return float(a @ (DX * DX) @ a + b @ (DY * DY) @ b - 2.0 * np.sum((DX @ T @ DY) * T))


def entropic_gw_2d(axis_x, axis_y, p, q, eps, outer, inner, k=1):
    """Entropic GW on 2-D grids: the same mirror-descent schedule as oracle.entropic_gw
    (Remark 1; readings R5, R7) with the 2-D gradient."""
    p, q = _f64(p), _f64(q)
    T = np.outer(p, q)
    f = np.zeros(p.size)
    g = np.zeros(q.size)
    out = {"E": [], "viol": []}
    for _ in range(outer):
        G = grad_prescribed_2d(axis_x, axis_y, p, q, T, k)
        f, g, _used = sinkhorn(G, p, q, eps, inner, f, g)
        T = plan_from_duals(G, f, g, eps)
        out["E"].append(objective_2d(axis_x, axis_y, T, k))
        out["viol"].append(violation(T, p, q))
    out.update(T=T, f=f, g=g, gw_objective=out["E"][-1] if outer else objective_2d(axis_x, axis_y, T, k))
    out["entropic_objective"] = out["gw_objective"] + eps * entropy(T)
    return out


def fgw_grad_prescribed_2d(axis_x, axis_y, p, q, fx, fy, alpha, T, k=1):
    """FGW gradient on 2-D grids (Remark 2, reading R29): per-point features
    fx (n), fy (m), C o C = (fx_i - fy_p)^2, theta = alpha:
        (1 - theta) C o C + theta * grad_prescribed_2d."""
    fx, fy = _f64(fx), _f64(fy)
    CC = (fx[:, None] - fy[None, :]) ** 2
    return (1.0 - alpha) * CC + alpha * grad_prescribed_2d(axis_x, axis_y, p, q, T, k)


def fgw_objective_2d(axis_x, axis_y, fx, fy, alpha, T, k=1):
    """E_bar(T) = (1 - theta) sum c_ip^2 T_ip + theta E(T)."""
    fx, fy, T = _f64(fx), _f64(fy), _f64(T)
    CC = (fx[:, None] - fy[None, :]) ** 2
    return float((1.0 - alpha) * np.sum(CC * T) + alpha * objective_2d(axis_x, axis_y, T, k))


def entropic_fgw_2d(axis_x, axis_y, p, q, fx, fy, alpha, eps, outer, inner, k=1):
    """Entropic FGW on 2-D grids: entropic_gw_2d's schedule with the FGW gradient (Remark 2)."""
    p, q = _f64(p), _f64(q)
    T = np.outer(p, q)
    f = np.zeros(p.size)
    g = np.zeros(q.size)
    out = {"E": [], "viol": []}
    for _ in range(outer):
        G = fgw_grad_prescribed_2d(axis_x, axis_y, p, q, fx, fy, alpha, T, k)
        f, g, _used = sinkhorn(G, p, q, eps, inner, f, g)
        T = plan_from_duals(G, f, g, eps)
        out["E"].append(fgw_objective_2d(axis_x, axis_y, fx, fy, alpha, T, k))
        out["viol"].append(violation(T, p, q))
    out.update(T=T, f=f, g=g, gw_objective=out["E"][-1])
    out["entropic_objective"] = out["gw_objective"] + eps * entropy(T)
    return out
