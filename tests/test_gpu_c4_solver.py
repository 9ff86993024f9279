"""C4 parity on the BENCHMARKED path (BASELINE.json configs[3]: N = M = 65536, eps = 1e-3, the
solver's own Gibbs-mode gradient kernels and fused Sinkhorn iterations, exactly as bench.py runs
them), SURVEY §8(c) C4 (ii) and (iii):

* per step: at outer iterations l in {1, 5, 10} the solver exports (gw_solve_set_export) the plan
  T^{l-1} its gradient is evaluated on and its own stored G^l; 64 random rows and 64 random columns
  of G^l are checked against c3 = 2(c 1^T + 1 c'^T) - 4 D_X T^{l-1} D_Y evaluated
  by the float64 oracle on those lines (oracle.grad_rows_cols), at <= 1e-5 max|G| (north_star);
* final plan (l = 10): the marginal violation from float64 host sums of the GPU's T and
  E(T_GPU) from the oracle's streamed k = 1 evaluation (oracle.objective_k1) against
  the GPU's reported values (objective <= 1e-4 relative, north_star).

Host memory: ~17 GB (the plan) + ~10 GB of float64 temporaries per worker; the GPU box has 196 GB.
"""

import os

import numpy as np
import pytest

import oracle as O
import workloads as W

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

N = 65536
BLK = 2048
GRAD_TOL = 1e-5
OBJ_TOL = 1e-4


@pytest.fixture(scope="module")
def c4():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as ge
    ge.build()
    from paper_2404_08970_b200 import api
    P = W.config4(N)
    return {"api": api, "P": P, "dev": torch.device("cuda", 0),
            "const": O.const_term_blocked(P.x, P.y, P.p, P.q)}


def _host_blocks(Tdev):
    """The plan on the host (fp32), as row-block views."""
    import torch
    Th = torch.empty(Tdev.shape, dtype=torch.float32, pin_memory=True)
    Th.copy_(Tdev)
    Tn = Th.numpy()
    return Tn, [(j, Tn[j:j + BLK]) for j in range(0, Tn.shape[0], BLK)]


@pytest.mark.parametrize("l", [1, 5, 10])
def test_c4_solver_gradient_step(c4, l):
    import torch
    api, P, dev = c4["api"], c4["P"], c4["dev"]
    Tb = api.plan_buffer(N, N, dev)
    Gb = api.plan_buffer(N, N, dev)
    r = api.solve(P.x, P.y, P.p, P.q, P.eps, l, P.inner, device=dev, export_iter=l, export_T=Tb, export_G=Gb)
    assert r.inner_fused_total > 0  # the benchmarked (fused) Sinkhorn path ran
    rng = np.random.default_rng(1000 + l)
    I = np.sort(rng.choice(N, 64, replace=False))
    J = np.sort(rng.choice(N, 64, replace=False))
    It = torch.from_numpy(I).to(dev)
    Jt = torch.from_numpy(J).to(dev)
    GI = Gb.index_select(0, It).cpu().numpy().astype(np.float64)
    GJ = Gb.index_select(1, Jt).cpu().numpy().astype(np.float64)
    del Gb
    _, blocks = _host_blocks(Tb)
    del Tb
    torch.cuda.empty_cache()
    OI, OJ = O.grad_rows_cols(P.x, P.y, P.p, P.q, blocks, I, J, const=c4["const"])
    scale = max(np.max(np.abs(OI)), np.max(np.abs(OJ)))
    err_r = np.max(np.abs(GI - OI)) / scale
    err_c = np.max(np.abs(GJ - OJ)) / scale
    print("C4 l=%d: gradient max-abs error / max|G|: rows %.3e, columns %.3e" % (l, err_r, err_c))
    assert err_r <= GRAD_TOL and err_c <= GRAD_TOL, (err_r, err_c)


def test_c4_final_plan_objective_and_violation(c4):
    import torch
    api, P, dev = c4["api"], c4["P"], c4["dev"]
    r = api.solve(P.x, P.y, P.p, P.q, P.eps, P.outer, P.inner, device=dev, return_plan=True)
    _, blocks = _host_blocks(r.T)
    r.T = None
    torch.cuda.empty_cache()
    viol = O.violation_streamed(blocks, P.p, P.q)
    workers = max(1, min(8, (os.cpu_count() or 2) // 2))
    E = O.objective_k1(P.x, P.y, blocks, workers=workers)
    rel = abs(r.gw_objective - E) / abs(E)
    print("C4 final: E_gpu %.10e E_oracle(T_gpu) %.10e rel %.3e; violation gpu %.3e host %.3e (N*viol %.3e)"
          % (r.gw_objective, E, rel, r.marginal_violation, viol, N * viol))
    assert rel <= OBJ_TOL
    # the GPU's reported violation describes its own plan (fp32 entries, fp64 sums on both sides)
    assert abs(r.marginal_violation - viol) <= 1e-8 + 0.02 * viol
    assert viol <= 1e-6  # north_star (absolute; R10)
