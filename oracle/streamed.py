"""Oracle evaluations for plans too large for dense N x N distance matrices (C4: N = M = 65536,
a 17 GB fp32 plan): the same definitions as oracle.gw, streamed over row blocks of T.
TEST INFRASTRUCTURE ONLY (tests/, smoke(), bench.py's cpu_baseline): the product path never
imports this package.

T is supplied as consecutive row blocks (j0, T[j0:j1]) (any float dtype; widened to float64 block
by block); objective_k1 iterates them twice, so it takes a sequence (e.g. views of a host array).

* grad_rows_cols: rows I and columns J of c3 = 2(c 1^T + 1 c'^T) - 4 D_X T D_Y (PAPER.md:120-126,
  reading R4: prescribed p, q), as SURVEY §8(c) C4 (ii) prescribes: rows by (D_X[I, :] T) D_Y,
  columns by D_X (T D_Y[:, J]); the N x |J| and |I| x M products are blocked DGEMMs with D
  generated blockwise, the remaining one-dimensional products are the paper's recursion
  (oracle.ref_dp_distance) batched over the sampled lines.
* objective_k1 / violation_streamed: E(T) = a^T (D_X o D_X) a + b^T (D_Y o D_Y) b
  - 2 <D_X T D_Y, T> with realised marginals (reading R13) and
  max(|T1 - p|_inf, |T^T 1 - q|_inf) for k = 1.  <D_X T D_Y, T> = <D_X T, T D_Y>
  with both factors formed by the k = 1 definition written as prefix sums,
      sum_j |s_i - s_j| v_j = s_i (P_<i - P_>i) - (Q_<i - Q_>i),  P = cumsum(v), Q = cumsum(s v),
  (distributivity of the lower / upper triangular sums), in float64.
* fgw_rows_cols / fgw_objective_k1 (C5: 32768 x 24576): Remark 2's gradient and objective
   from the GW pieces above and the feature cost (fx_i - fy_p)^2 (reading R29).
* ugw_functional_k1: F_eps of reading R33 (PAPER.md:150-153 + the entropic term) for a streamed plan:
  E by objective_k1, the three tensorised KLs by KL(x (x) x | y (x) y) = 2 m(x) <log(x/y), x> - m(x)^2
  + m(y)^2 with the plan's <log(T/(u v)), T> accumulated block by block (0 log 0 = 0).
"""

import numpy as np

from .gw import _f64, ref_dp_distance

__all__ = ["const_term_blocked", "grad_rows_cols", "marginals_streamed", "violation_streamed",
           "objective_k1", "dist_apply_prefix", "fgw_rows_cols", "fgw_objective_k1", "ugw_functional_k1"]

BLK = 2048


def const_term_blocked(x, y, p, q, k=1, block=BLK):
    """(c, c') = ((D_X o D_X) p, (D_Y o D_Y) q) (reading R3), rows of the dense
    definition generated block by block."""
    def one(s, w):
        s, w = _f64(s), _f64(w)
        out = np.empty(s.size)
        for b in range(0, s.size, block):
            out[b:b + block] = (np.abs(s[b:b + block, None] - s[None, :]) ** (2 * k)) @ w
        return out
    return one(x, p), one(y, q)


def grad_rows_cols(x, y, p, q, T_blocks, I, J, k=1, const=None):
    """Rows I (|I| x M) and columns J (N x |J|) of c3 on a streamed plan (see module doc).
    const: (c, c') from const_term_blocked, if already computed."""
    x, y = _f64(x), _f64(y)
    I, J = np.asarray(I), np.asarray(J)
    n, m = x.size, y.size
    U = np.zeros((I.size, m))          # D_X[I, :] T
    V = np.zeros((n, J.size))          # T D_Y[:, J]
    DYJ = np.abs(y[:, None] - y[None, J]) ** k
    seen = 0
    for j0, Tb in T_blocks:
        Tb = _f64(Tb)
        j1 = j0 + Tb.shape[0]
        U += (np.abs(x[I, None] - x[None, j0:j1]) ** k) @ Tb
        V[j0:j1] = Tb @ DYJ
        seen += Tb.shape[0]
    if seen != n:
        raise ValueError("grad_rows_cols: the row blocks cover %d of %d rows" % (seen, n))
    R = ref_dp_distance(U, y, k)               # (D_X[I, :] T) D_Y, row by row (D_Y symmetric)
    Cc = ref_dp_distance(V.T, x, k).T          # D_X (T D_Y[:, J]), column by column
    c, c2 = const if const is not None else const_term_blocked(x, y, p, q, k)
    GI = 2.0 * (c[I, None] + c2[None, :]) - 4.0 * R
    GJ = 2.0 * (c[:, None] + c2[None, J]) - 4.0 * Cc
    return GI, GJ


def marginals_streamed(T_blocks, n, m):
    """Realised marginals a = T 1 (n), b = T^T 1 (m) in float64."""
    a = np.zeros(n)
    b = np.zeros(m)
    for j0, Tb in T_blocks:
        Tb = _f64(Tb)
        a[j0:j0 + Tb.shape[0]] = Tb.sum(axis=1)
        b += Tb.sum(axis=0)
    return a, b


def violation_streamed(T_blocks, p, q):
    """max(||T1 - p||_inf, ||T^T 1 - q||_inf), float64 sums (reading R10)."""
    p, q = _f64(p), _f64(q)
    a, b = marginals_streamed(T_blocks, p.size, q.size)
    return float(max(np.max(np.abs(a - p)), np.max(np.abs(b - q))))


def dist_apply_prefix(v, s, axis=-1):
    """D v along `axis` for D_ij = |s_i - s_j| (k = 1) by prefix sums (module doc)."""
    v = np.moveaxis(_f64(v), axis, -1)
    s = _f64(s)
    P = np.cumsum(v, axis=-1)
    Q = np.cumsum(v * s, axis=-1)
    Pt, Qt = P[..., -1:], Q[..., -1:]
    # sum_{j<=i}: inclusive sums; the j = i term has |s_i - s_i| = 0 so inclusive == exclusive
    out = s * (2.0 * P - Pt) - (2.0 * Q - Qt)
    return np.moveaxis(out, -1, axis)


def objective_k1(x, y, T_blocks, workers=1):
    """E(T) (k = 1) for a streamed plan (module doc).  T_blocks: a sequence of (j0, block) that can
    be iterated twice (e.g. a list of views of a host array).

    Pass 1: realised marginals a, b, the column moments b_x = T^T x (for the suffix sums of D_X T)
    and every block's column sums (its carry-in is the exclusive prefix over the blocks above).
    Pass 2: per row block, W = T D_Y (row-local) and V = D_X T (column prefix sums from the
    carry-in plus the block's own cumulative sums, suffixes from the totals); accumulate <V, W>.
    The blocks of pass 2 are independent, so they may run on a thread pool (NumPy releases the
    GIL); the per-block sums are added in block order."""
    from concurrent.futures import ThreadPoolExecutor
    x, y = _f64(x), _f64(y)
    n, m = x.size, y.size
    blocks = list(T_blocks)

    def moments(item):
        j0, Tb = item
        Tb = _f64(Tb)
        j1 = j0 + Tb.shape[0]
        return Tb.sum(axis=1), Tb.sum(axis=0), x[j0:j1] @ Tb

    def run(fn, items):
        if workers > 1:
            with ThreadPoolExecutor(workers) as ex:
                return list(ex.map(fn, items))
        return [fn(it) for it in items]

    mom = run(moments, blocks)
    a = np.zeros(n)
    b = np.zeros(m)
    bx = np.zeros(m)
    carry = []
    for (j0, Tb), (ra, cb, cbx) in zip(blocks, mom):
        carry.append((b.copy(), bx.copy()))   # exclusive prefix over the blocks above
        a[j0:j0 + ra.size] = ra
        b += cb
        bx += cbx
    if a.size != n or sum(Tb.shape[0] for _, Tb in blocks) != n:
        raise ValueError("objective_k1: the row blocks do not cover the plan")

    def cross(args):
        (j0, Tb), (Pc, Qc) = args
        Tb = _f64(Tb)
        xb = x[j0:j0 + Tb.shape[0], None]
        W = dist_apply_prefix(Tb, y, axis=1)                       # (T D_Y) rows of the block
        P = Pc[None, :] + np.cumsum(Tb, axis=0)                    # inclusive column prefix, all rows
        Q = Qc[None, :] + np.cumsum(xb * Tb, axis=0)
        V = xb * (2.0 * P - b[None, :]) - (2.0 * Q - bx[None, :])  # (D_X T) rows of the block
        return float(np.sum(V * W))

    total = 0.0
    for v in run(cross, list(zip(blocks, carry))):
        total += v

    # a^T (D_X o D_X) a = sum_ij (x_i - x_j)^2 a_i a_j, expanded in moments of a (k = 1)
    def quad(s, w):
        m0, m1, m2 = w.sum(), w @ s, w @ (s * s)
        return 2.0 * (m0 * m2 - m1 * m1)
    return float(quad(x, a) + quad(y, b) - 2.0 * total)


def fgw_rows_cols(x, y, p, q, fx, fy, alpha, T_blocks, I, J, const=None):
    """Rows I and columns J of grad E_bar = (1 - theta) C o C + theta (2(c 1^T + 1 c'^T) - 4 D_X T D_Y)
    (PAPER.md:141-145 with theta = alpha, transpose typo fixed as in R3; C o C = (fx_i - fy_p)^2)."""
    fx, fy = _f64(fx), _f64(fy)
    I, J = np.asarray(I), np.asarray(J)
    GI, GJ = grad_rows_cols(x, y, p, q, T_blocks, I, J, 1, const)
    return ((1.0 - alpha) * (fx[I, None] - fy[None, :]) ** 2 + alpha * GI,
            (1.0 - alpha) * (fx[:, None] - fy[None, J]) ** 2 + alpha * GJ)


def fgw_objective_k1(x, y, fx, fy, alpha, T_blocks, workers=1):
    """E_bar(T) = (1 - theta) sum_ip (fx_i - fy_p)^2 T_ip + theta E(T), streamed."""
    fx, fy = _f64(fx), _f64(fy)
    blocks = list(T_blocks)
    lin = 0.0
    for j0, Tb in blocks:
        Tb = _f64(Tb)
        lin += float(np.sum((fx[j0:j0 + Tb.shape[0], None] - fy[None, :]) ** 2 * Tb))
    return (1.0 - alpha) * lin + alpha * objective_k1(x, y, blocks, workers)


def ugw_functional_k1(x, y, u, v, T_blocks, rho, eps, workers=1):
    """F_eps(G) (reading R33) for a streamed plan, k = 1.  Returns (F, E, mass)."""
    u, v = _f64(u), _f64(v)
    blocks = list(T_blocks)
    a, b = marginals_streamed(blocks, u.size, v.size)

    def xlogy_sum(w, ref):       # <log(w/ref), w>, 0 log 0 = 0
        pos = w > 0
        return float(np.sum(w[pos] * np.log(w[pos] / ref[pos])))

    def kl_sq(w, ref):           # KL(w (x) w | ref (x) ref)
        return 2.0 * w.sum() * xlogy_sum(w, ref) - w.sum() ** 2 + ref.sum() ** 2

    ent = 0.0
    for j0, Tb in blocks:
        Tb = _f64(Tb)
        ent += xlogy_sum(Tb, u[j0:j0 + Tb.shape[0], None] * v[None, :])
    mass = float(a.sum())
    kl_plan = 2.0 * mass * ent - mass ** 2 + (u.sum() * v.sum()) ** 2
    E = objective_k1(x, y, blocks, workers)
    return E + rho * kl_sq(a, u) + rho * kl_sq(b, v) + eps * kl_plan, E, mass
