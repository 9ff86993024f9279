"""GPU parity for 2-D grids (Table 3): the GW_GRID2D path
through the C ABI against oracle/grid2d.py on the same seeded inputs.  Tolerances as in
test_gpu_parity.py (BASELINE.json north_star).
"""

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

GRAD_TOL = 1e-5
OBJ_TOL = 1e-4
VIOL_TOL = 1e-6


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


def _err(G, Go):
    return np.max(np.abs(G - Go)) / max(np.max(np.abs(Go)), 1e-300)


def _axis(rng, n, uniform):
    """Uniform grid s_a = a h (the paper's Table 3 grid) or a sorted random axis with a tie."""
    if uniform:
        return np.arange(n) / max(n - 1.0, 1.0)
    s = np.sort(rng.random(n))
    if n > 3:
        s[2] = s[1]
    return s


def _problem(seed, nx, ny, uniform=True):
    """Table-3 style input: grid supports, U[0,1] weights normalised."""
    rng = np.random.default_rng(seed)
    sx, sy = _axis(rng, nx, uniform), _axis(rng, ny, uniform)
    p, q = rng.random(nx * nx) + 0.05, rng.random(ny * ny) + 0.05
    return rng, sx, sy, p / p.sum(), q / q.sum()


@pytest.mark.parametrize("nx,ny,uniform", [(1, 1, True), (1, 3, True), (2, 3, False), (4, 4, True), (8, 5, False),
                                           (16, 16, True), (33, 20, False), (20, 33, True)])
def test_grad_2d_random_plan(gw, nx, ny, uniform):
    """gw_grad_dp with GW_GRID2D vs oracle.grad_prescribed_2d (dense definition) on a random plan."""
    rng, sx, sy, p, q = _problem(nx * 100 + ny, nx, ny, uniform)
    T = (rng.exponential(size=(nx * nx, ny * ny)) / (nx * nx * ny * ny)).astype(np.float32)
    G = gw.grad(sx, sy, p, q, _to_dev(gw, T), grid2d=True).cpu().numpy().astype(np.float64)
    Go = O.grad_prescribed_2d(sx, sy, p, q, T.astype(np.float64))
    assert _err(G, Go) <= GRAD_TOL


def test_grad_2d_64x48_full(gw):
    """N = 4096, M = 2304 (spans many CTAs), full matrix vs the dense oracle."""
    rng, sx, sy, p, q = _problem(7, 64, 48, True)
    T = (rng.random((64 * 64, 48 * 48)) / (64 * 64 * 48 * 48)).astype(np.float32)
    G = gw.grad(sx, sy, p, q, _to_dev(gw, T), grid2d=True).cpu().numpy().astype(np.float64)
    Go = O.grad_prescribed_2d(sx, sy, p, q, T.astype(np.float64))
    assert _err(G, Go) <= GRAD_TOL


def test_grad_2d_max_side(gw):
    """nx = 256 (N = 65536 rows, the largest grid the path takes) x ny = 16: every row against the
    oracle's Kronecker product (apply_distance_2d, pinned to the dense definition)."""
    rng, sx, sy, p, q = _problem(11, 256, 16, False)
    n, m = 256 * 256, 16 * 16
    T = (rng.random((n, m)) / (n * m)).astype(np.float32)
    G = gw.grad(sx, sy, p, q, _to_dev(gw, T), grid2d=True).cpu().numpy().astype(np.float64)
    T64 = T.astype(np.float64)
    DXT = np.stack([O.apply_distance_2d(T64[:, j], sx) for j in range(m)], axis=1)   # D_X T
    DYf = O.dist2d(sy)
    c2 = (DYf * DYf) @ q
    P = O.grid_points(sx)
    for i in rng.choice(n, 64, replace=False):
        di = np.abs(P[i, 0] - P[:, 0]) + np.abs(P[i, 1] - P[:, 1])
        Go = 2.0 * (np.sum(di * di * p) + c2) - 4.0 * O.apply_distance_2d(DXT[i], sy)
        assert np.max(np.abs(G[i] - Go)) <= GRAD_TOL * np.max(np.abs(Go)), i


def _grad_2d_rows_oracle(sx, sy, p, q, T64, rows):
    """Rows of the 2-D gradient by the oracle's Kronecker products (apply_distance_2d, pinned to the
    dense definition): W = T D_Y row by row, then (D_X W)_i with the dense D_X."""
    W = np.stack([O.apply_distance_2d(T64[j], sy) for j in range(T64.shape[0])])  # T D_Y (D_Y symmetric)
    DX = O.dist2d(sx)
    Px, Py = O.grid_points(sx), O.grid_points(sy)
    out = []
    for i in rows:
        dxi = np.abs(Px[i, 0] - Px[:, 0]) + np.abs(Px[i, 1] - Px[:, 1])
        c_i = np.sum(dxi * dxi * p)
        out.append((i, c_i, DX[i] @ W))
    DYq = np.array([np.sum((np.abs(Py[j, 0] - Py[:, 0]) + np.abs(Py[j, 1] - Py[:, 1])) ** 2 * q)
                    for j in range(Py.shape[0])])
    return {i: 2.0 * (c_i + DYq) - 4.0 * v for i, c_i, v in out}


@pytest.mark.parametrize("nx,ny", [(8, 128), (6, 256)])
def test_grad_2d_wide_rows(gw, nx, ny):
    """Rows of 128^2 / 256^2 columns take the 128-bit reduction kernel (k_g2_rowred4): every row vs the
    oracle's Kronecker route."""
    rng, sx, sy, p, q = _problem(5 * nx + ny, nx, ny, False)
    n, m = nx * nx, ny * ny
    T = (rng.random((n, m)) / (n * m)).astype(np.float32)
    G = gw.grad(sx, sy, p, q, _to_dev(gw, T), grid2d=True).cpu().numpy().astype(np.float64)
    ref = _grad_2d_rows_oracle(sx, sy, p, q, T.astype(np.float64), range(n))
    scale = max(np.max(np.abs(v)) for v in ref.values())
    err = max(np.max(np.abs(G[i] - v)) for i, v in ref.items()) / scale
    print("2-D wide rows nx=%d ny=%d: gradient err / max|G| %.3e" % (nx, ny, err))
    assert err <= GRAD_TOL


def test_solver_2d_wide_rows_gibbs_gradient(gw, monkeypatch):
    """The solver's own gradient on a Gibbs plan (T^1 regenerated from G^1 and the duals) through the
    128-bit reduction kernel: exported G^2 vs the oracle on the exported T^1; and the whole solve with
    the scalar kernel (GWDP_G2_SCALAR=1) agrees."""
    _, sx, sy, p, q = _problem(77, 12, 128, False)
    n, m = 144, 128 * 128
    Tb, Gb = gw.plan_buffer(n, m, _dev()), gw.plan_buffer(n, m, _dev())
    r = gw.solve(sx, sy, p, q, 0.01, 2, 50, device=_dev(), grid2d=True, export_iter=2, export_T=Tb, export_G=Gb)
    T64 = Tb.cpu().numpy().astype(np.float64)
    G = Gb.cpu().numpy().astype(np.float64)
    rows = np.random.default_rng(0).choice(n, 24, replace=False)
    ref = _grad_2d_rows_oracle(sx, sy, p, q, T64, rows)
    scale = max(np.max(np.abs(v)) for v in ref.values())
    err = max(np.max(np.abs(G[i] - v)) for i, v in ref.items()) / scale
    monkeypatch.setenv("GWDP_G2_SCALAR", "1")
    r2 = gw.solve(sx, sy, p, q, 0.01, 2, 50, device=_dev(), grid2d=True)
    rel = abs(r.gw_objective - r2.gw_objective) / abs(r2.gw_objective)
    print("2-D Gibbs gradient err / max|G| %.3e; objective vector vs scalar kernel %.3e" % (err, rel))
    assert err <= GRAD_TOL
    assert rel <= 1e-5


def test_grad_2d_product_plan_closed_form(gw):
    """T = p q^T: D_X T D_Y = (D_X p)(D_Y q)^T, each factor by the oracle's dense D."""
    rng, sx, sy, p, q = _problem(3, 12, 9, False)
    T = np.outer(p, q)
    G = gw.grad(sx, sy, p, q, _to_dev(gw, T), grid2d=True).cpu().numpy().astype(np.float64)
    DX, DY = O.dist2d(sx), O.dist2d(sy)
    Go = 2.0 * (((DX * DX) @ p)[:, None] + ((DY * DY) @ q)[None, :]) - 4.0 * np.outer(DX @ p, DY @ q)
    assert _err(G, Go) <= GRAD_TOL


@pytest.mark.parametrize("nx,ny,eps", [(8, 6, 0.02), (16, 12, 0.01), (24, 24, 0.005)])
def test_solver_2d_trajectory(gw, nx, ny, eps):
    """entropic_gw_solve with GW_GRID2D vs oracle.entropic_gw_2d: objective trajectory, final
    objective, entropic objective and violation."""
    _, sx, sy, p, q = _problem(nx + 31 * ny, nx, ny, True)
    outer, inner = 5, 100
    r = gw.solve(sx, sy, p, q, eps, outer, inner, trace_objective=True, return_plan=True, device=_dev(),
                 grid2d=True)
    ro = O.entropic_gw_2d(sx, sy, p, q, eps, outer, inner)
    E = np.asarray(ro["E"])
    assert np.max(np.abs(r.trace[:, 0] - E) / np.abs(E)) <= OBJ_TOL
    assert abs(r.gw_objective - ro["gw_objective"]) <= OBJ_TOL * abs(ro["gw_objective"])
    assert abs(r.entropic_objective - ro["entropic_objective"]) <= OBJ_TOL * abs(ro["entropic_objective"])
    assert r.marginal_violation <= max(VIOL_TOL, 2 * ro["viol"][-1])
    T = r.T.cpu().numpy().astype(np.float64)
    assert abs(O.objective_2d(sx, sy, T) - r.gw_objective) <= OBJ_TOL * abs(r.gw_objective)


@pytest.mark.parametrize("alpha", [0.5, 1.0])
def test_fgw_solver_2d(gw, alpha):
    """fgw_solve with GW_GRID2D vs oracle.entropic_fgw_2d (Remark 2)."""
    rng, sx, sy, p, q = _problem(21, 10, 8, False)
    fx, fy = rng.random(100), rng.random(64)
    r = gw.solve(sx, sy, p, q, 0.02, 4, 80, fx=fx, fy=fy, alpha=alpha, trace_objective=True, device=_dev(),
                 grid2d=True)
    ro = O.entropic_fgw_2d(sx, sy, p, q, fx, fy, alpha, 0.02, 4, 80)
    E = np.asarray(ro["E"])
    assert np.max(np.abs(r.trace[:, 0] - E) / np.abs(E)) <= OBJ_TOL
    assert abs(r.gw_objective - ro["gw_objective"]) <= OBJ_TOL * abs(ro["gw_objective"])


def test_solver_2d_host_vectors_match_device(gw):
    _, sx, sy, p, q = _problem(5, 9, 7, False)
    a = gw.solve(sx, sy, p, q, 0.02, 3, 50, device=_dev(), grid2d=True)
    b = gw.solve_host(sx, sy, p, q, 0.02, 3, 50, grid2d=True)
    assert a.gw_objective == b.gw_objective
    np.testing.assert_array_equal(a.f.cpu().numpy(), b.f)


def test_grid2d_errors(gw):
    from paper_2404_08970_b200 import GwError, _lib as L
    import ctypes as C
    import torch
    _, sx, sy, p, q = _problem(1, 4, 4, True)
    T = _to_dev(gw, np.full((16, 16), 1 / 256, dtype=np.float32))
    with pytest.raises(GwError) as e:  # k = 2 on grids
        gw.grad(sx, sy, p, q, T, k=2, grid2d=True)
    assert e.value.code == "GW_ERR_UNSUPPORTED"
    with pytest.raises(GwError) as e:  # unsorted axis
        gw.grad(sx[::-1].copy(), sy, p, q, T, grid2d=True)
    assert e.value.code == "GW_ERR_UNSORTED"
    with pytest.raises(ValueError):
        gw.grad(sx, sy, p[:15], q, T, grid2d=True)
    # n not a perfect square -> INVALID_ARG from the library itself
    ctx = gw.Context.get(_dev())
    dev = _dev()
    xs = torch.tensor(sx, device=dev)
    pp = torch.full((15,), 1 / 15, dtype=torch.float64, device=dev)
    pr = gw._problem(xs, xs, pp, torch.tensor(q, device=dev))
    pr.n, pr.n_local, pr.m, pr.flags = 15, 15, 16, L.GW_GRID2D
    Tb = gw.plan_buffer(15, 16, dev)
    with pytest.raises(GwError) as e:
        L.check(ctx.lib.gw_grad_dp(ctx.h, C.byref(pr), Tb.data_ptr(), Tb.stride(0), Tb.data_ptr(), Tb.stride(0), None))
    assert e.value.code == "GW_ERR_INVALID_ARG"
    # side > 256
    ax = np.arange(257) / 256.0
    pw = np.full(257 * 257, 1.0 / (257 * 257))
    Tb = gw.plan_buffer(257 * 257, 1, dev)
    with pytest.raises(GwError) as e:
        gw.grad(ax, [0.0], pw, [1.0], Tb, grid2d=True)
    assert e.value.code == "GW_ERR_UNSUPPORTED"
