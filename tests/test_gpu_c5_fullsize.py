"""C5 at FULL size (BASELINE.json configs[4]: N = 32768, M = 24576, supports ~ Beta(2,5) / Beta(5,2),
feature cost (f_i - g_j)^2, alpha = 0.5, Dirichlet(0.5) marginals, KL-unbalanced rho = 1.0), on the
solver paths the C5 timings in profiles/ come from (K = 6 fused clusters, FGW term fused into the
gradient kernels, UGW on the fused iteration):

* FGW per step: at outer iterations l in {1, 2, 5} the solver exports (gw_solve_set_export) the plan
  T^{l-1} and its own stored cost G^l = grad E_bar(T^{l-1}); 48 random rows + 48 random columns are
  checked against PAPER.md:141-145 evaluated by the float64 oracle on those lines
  (oracle.fgw_rows_cols), at <= 1e-5 max|G| (north_star);
* FGW final plan (20 x 100): E_bar(T_GPU) by oracle.fgw_objective_k1 and the
  two-sided violation from float64 host sums, against the GPU's reported values;
* UGW final plan (3 x 100, rho = 1): F_eps, E and the mass of the GPU's plan by
  oracle.ugw_functional_k1 (reading R33) against the GPU's reported values.

Host memory: 3.2 GB (the fp32 plan) + float64 temporaries per worker.
"""

import os

import numpy as np
import pytest

import oracle as O
import workloads as W

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

BLK = 2048
GRAD_TOL = 1e-5
OBJ_TOL = 1e-4


@pytest.fixture(scope="module")
def c5():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as ge
    ge.build()
    from paper_2404_08970_b200 import api
    P = W.config5()
    assert (P.x.size, P.y.size) == (32768, 24576)
    return {"api": api, "P": P, "dev": torch.device("cuda", 0),
            "const": O.const_term_blocked(P.x, P.y, P.p, P.q),
            "workers": max(1, min(8, (os.cpu_count() or 2) // 2))}


def _host_blocks(Tdev):
    import torch
    Th = torch.empty(Tdev.shape, dtype=torch.float32, pin_memory=True)
    Th.copy_(Tdev)
    Tn = Th.numpy()
    return Tn, [(j, Tn[j:j + BLK]) for j in range(0, Tn.shape[0], BLK)]


@pytest.mark.parametrize("l", [1, 2, 5])
def test_c5_fgw_solver_gradient_step(c5, l):
    import torch
    api, P, dev = c5["api"], c5["P"], c5["dev"]
    n, m = P.x.size, P.y.size
    Tb = api.plan_buffer(n, m, dev)
    Gb = api.plan_buffer(n, m, dev)
    r = api.solve(P.x, P.y, P.p, P.q, P.eps, l, P.inner, fx=P.fx, fy=P.fy, alpha=P.alpha, device=dev,
                  export_iter=l, export_T=Tb, export_G=Gb)
    if l > 1:
        assert r.inner_fused_total > 0  # the fused one-read Sinkhorn path ran
    rng = np.random.default_rng(2000 + l)
    I = np.sort(rng.choice(n, 48, replace=False))
    J = np.sort(rng.choice(m, 48, replace=False))
    GI = Gb.index_select(0, torch.from_numpy(I).to(dev)).cpu().numpy().astype(np.float64)
    GJ = Gb.index_select(1, torch.from_numpy(J).to(dev)).cpu().numpy().astype(np.float64)
    del Gb
    _, blocks = _host_blocks(Tb)
    del Tb
    torch.cuda.empty_cache()
    OI, OJ = O.fgw_rows_cols(P.x, P.y, P.p, P.q, P.fx, P.fy, P.alpha, blocks, I, J, const=c5["const"])
    scale = max(np.max(np.abs(OI)), np.max(np.abs(OJ)))
    err_r = np.max(np.abs(GI - OI)) / scale
    err_c = np.max(np.abs(GJ - OJ)) / scale
    print("C5 FGW l=%d: gradient max-abs error / max|G|: rows %.3e, columns %.3e (max|G| %.3e)"
          % (l, err_r, err_c, scale))
    assert err_r <= GRAD_TOL and err_c <= GRAD_TOL, (err_r, err_c)


def test_c5_fgw_final_plan_objective_and_violation(c5):
    import torch
    api, P, dev = c5["api"], c5["P"], c5["dev"]
    r = api.solve(P.x, P.y, P.p, P.q, P.eps, P.outer, P.inner, fx=P.fx, fy=P.fy, alpha=P.alpha, device=dev,
                  return_plan=True)
    _, blocks = _host_blocks(r.T)
    r.T = None
    torch.cuda.empty_cache()
    viol = O.violation_streamed(blocks, P.p, P.q)
    Eb = O.fgw_objective_k1(P.x, P.y, P.fx, P.fy, P.alpha, blocks, workers=c5["workers"])
    rel = abs(r.gw_objective - Eb) / abs(Eb)
    print("C5 FGW final (%d x %d): E_bar gpu %.10e oracle(T_gpu) %.10e rel %.3e; violation gpu %.3e host %.3e"
          % (P.outer, P.inner, r.gw_objective, Eb, rel, r.marginal_violation, viol))
    assert rel <= OBJ_TOL
    assert abs(r.marginal_violation - viol) <= 1e-8 + 0.02 * viol
    assert viol <= 1e-6  # north_star (absolute; R10)


def test_c5_ugw_final_plan_functional(c5):
    import torch
    api, P, dev = c5["api"], c5["P"], c5["dev"]
    outer = 3
    r = api.ugw_solve(P.x, P.y, P.p, P.q, P.rho, P.eps, outer, P.inner, trace_objective=True, return_plan=True,
                      device=dev)
    _, blocks = _host_blocks(r.T)
    r.T = None
    torch.cuda.empty_cache()
    F, E, mass = O.ugw_functional_k1(P.x, P.y, P.p, P.q, blocks, P.rho, P.eps, workers=c5["workers"])
    rel_F = abs(r.entropic_objective - F) / abs(F)
    rel_E = abs(r.gw_objective - E) / abs(E)
    m_gpu = float(r.trace[outer - 1, 3])
    print("C5 UGW final (%d x %d, rho %.1f): F gpu %.10e oracle(T_gpu) %.10e rel %.3e; E gpu %.10e oracle %.10e "
          "rel %.3e; mass gpu %.10f host %.10f" % (outer, P.inner, P.rho, r.entropic_objective, F, rel_F,
                                                   r.gw_objective, E, rel_E, m_gpu, mass))
    assert rel_F <= OBJ_TOL and rel_E <= OBJ_TOL
    assert abs(m_gpu - mass) <= 1e-6 * mass
    assert 0.0 < mass < 1.0 + 1e-6
