"""GPU parity of the solver's one-read DP gradient (8 N M bytes; csrc/rowclu.cuh):
the cost G^l the solver stores after a gradient on that path is exported (gw_solve_set_export)
together with the plan T^{l-1} it was evaluated on, and compared with the float64 oracle
c3 = 2(c 1^T + 1 c'^T) - 4 D_X T D_Y on that plan, at 1e-5 max|G| (north_star).

Shapes span every cluster width of the path (1, 2, 4, 8 and 16 CTAs of 4096 columns per row),
ragged M (M % 4 != 0, idle CTAs), fewer rows than clusters, and ties in the supports.  The whole
solve is also compared with the two-read path (GWDP_NO_RC=1) and, for a small case, with the
oracle's solve.
"""

import os

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

GRAD_TOL = 1e-5
OBJ_TOL = 1e-4


@pytest.fixture(scope="module")
def gw():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as ge
    ge.build()
    from paper_2404_08970_b200 import api
    # small shapes would otherwise run the whole inner loop in one cluster-resident launch (small.cuh)
    os.environ["GWDP_NO_SMALL"] = "1"
    os.environ["GWDP_RC"] = "1"
    yield api
    os.environ.pop("GWDP_NO_SMALL", None)
    os.environ.pop("GWDP_RC", None)


def _dev():
    import torch
    return torch.device("cuda", 0)


def _problem(seed, n, m):
    rng = np.random.default_rng(seed)
    x, y = np.sort(rng.random(n)), np.sort(rng.random(m))
    if n > 4:
        x[3] = x[2]  # ties
    if m > 4:
        y[1] = y[0]
    p, q = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
    return x, y, p, q


def _export(gw, x, y, p, q, eps, outer, inner, l):
    n, m = len(x), len(y)
    Tb = gw.plan_buffer(n, m, _dev())
    Gb = gw.plan_buffer(n, m, _dev())
    r = gw.solve(x, y, p, q, eps, outer, inner, device=_dev(), export_iter=l, export_T=Tb, export_G=Gb)
    return r, Tb, Gb


def _lines(n, m, rng, nr=48, nc=48):
    I = set([0, 1, n // 2, n - 1]) | set(rng.choice(n, min(n, nr), replace=False).tolist())
    J = set([0, m - 1]) | set(rng.choice(m, min(m, nc), replace=False).tolist())
    for b in range(4096, m, 4096):  # CTA boundaries of the 4096-column slices
        J |= {b - 1, b}
    return np.array(sorted(i for i in I if 0 <= i < n)), np.array(sorted(j for j in J if 0 <= j < m))


@pytest.mark.parametrize("n,m", [(300, 517), (1000, 4096), (777, 5003), (513, 16421), (96, 40000), (3, 300),
                                 (2500, 8192)])
def test_onepass_gradient_vs_oracle(gw, n, m):
    import torch
    x, y, p, q = _problem(n * 7 + m, n, m)
    eps = 0.02
    r, Tb, Gb = _export(gw, x, y, p, q, eps, 3, 20, 3)
    assert r.inner_fused_total > 0
    assert r.grad_onepass_total == 2, r.grad_onepass_total  # l = 2, 3 (l = 1: the product plan)
    T = Tb.cpu().numpy().astype(np.float64)
    G = Gb.cpu().numpy().astype(np.float64)
    if n * m <= 4_000_000 and max(n, m) <= 8192:
        Go = O.grad_prescribed(x, y, p, q, T)
        err = np.max(np.abs(G - Go)) / np.max(np.abs(Go))
        print("one-pass gradient %dx%d: max-abs error / max|G| = %.3e" % (n, m, err))
        assert err <= GRAD_TOL, err
    else:
        I, J = _lines(n, m, np.random.default_rng(n + m))
        blocks = [(j, T[j:j + 256]) for j in range(0, n, 256)]
        OI, OJ = O.grad_rows_cols(x, y, p, q, blocks, I, J)
        scale = max(np.max(np.abs(OI)), np.max(np.abs(OJ)))
        err_r = np.max(np.abs(G[I] - OI)) / scale
        err_c = np.max(np.abs(G[:, J] - OJ)) / scale
        print("one-pass gradient %dx%d: rows %.3e, columns %.3e of max|G|" % (n, m, err_r, err_c))
        assert err_r <= GRAD_TOL and err_c <= GRAD_TOL, (err_r, err_c)
    del Tb, Gb
    torch.cuda.empty_cache()


def test_onepass_solve_matches_two_read_path_and_oracle(gw):
    x, y, p, q = _problem(11, 400, 1300)
    eps, outer, inner = 0.02, 6, 40
    r1 = gw.solve(x, y, p, q, eps, outer, inner, device=_dev())
    os.environ["GWDP_NO_RC"] = "1"
    try:
        r0 = gw.solve(x, y, p, q, eps, outer, inner, device=_dev())
    finally:
        os.environ.pop("GWDP_NO_RC", None)
    assert r1.grad_onepass_total == outer - 1 and r0.grad_onepass_total == 0
    ro = O.entropic_gw(x, y, p, q, eps, outer, inner)
    rel1 = abs(r1.gw_objective - ro["gw_objective"]) / abs(ro["gw_objective"])
    rel0 = abs(r0.gw_objective - ro["gw_objective"]) / abs(ro["gw_objective"])
    print("solve: one-pass rel %.3e, two-read rel %.3e vs the oracle" % (rel1, rel0))
    assert rel1 <= OBJ_TOL and rel0 <= OBJ_TOL
    assert abs(r1.gw_objective - r0.gw_objective) <= 1e-5 * abs(r0.gw_objective)
    assert r1.marginal_violation <= 1e-6


def test_onepass_not_taken_where_unsupported(gw):
    """Tolerance rule, traced objective, FGW, k = 2: the two-read path (the XM sweep is not run)."""
    x, y, p, q = _problem(5, 200, 300)
    r = gw.solve(x, y, p, q, 0.02, 3, 40, tol=1e-7, check_every=10, device=_dev())
    assert r.grad_onepass_total == 0
    r = gw.solve(x, y, p, q, 0.02, 3, 40, trace_objective=True, device=_dev())
    assert r.grad_onepass_total == 0
    r = gw.solve(x, y, p, q, 0.02, 3, 40, k=2, device=_dev())
    assert r.grad_onepass_total == 0


@pytest.mark.parametrize("n,m", [(1, 1), (5, 300), (300, 517), (777, 5003), (2048, 1031)])
def test_product_plan_gradient_closed_form(gw, n, m):
    """The first outer iteration's gradient on T^0 = p q^T: the solver writes the closed form
    2c_i + 2c'_p - 4 (D_X p)_i (D_Y q)_p (k_grad_product); exported G^1 vs the oracle on p q^T."""
    x, y, p, q = _problem(n + 3 * m, n, m)
    r, Tb, Gb = _export(gw, x, y, p, q, 0.02, 1, 10, 1)
    T = Tb.cpu().numpy().astype(np.float64)
    np.testing.assert_allclose(T, np.outer(p, q), rtol=2e-7, atol=1e-30)
    G = Gb.cpu().numpy().astype(np.float64)
    Go = O.grad_prescribed(x, y, p, q, np.outer(p, q))
    err = np.max(np.abs(G - Go)) / max(np.max(np.abs(Go)), 1e-300)
    print("product-plan gradient %dx%d: %.3e of max|G|" % (n, m, err))
    assert err <= GRAD_TOL, err
