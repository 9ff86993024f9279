#!/usr/bin/env python
"""SURVEY §4.2 tier T5: a small workload touching every kernel family, to run under
compute-sanitizer (memcheck / racecheck / synccheck):

    compute-sanitizer --tool memcheck --error-exitcode 1 python scripts/sanitize.py
    compute-sanitizer --tool racecheck --error-exitcode 1 python scripts/sanitize.py
    compute-sanitizer --tool synccheck --error-exitcode 1 python scripts/sanitize.py

Sizes are small and ragged (several tiles, tails, m % 4 != 0).  Prints "sanitize workload ok".
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    from paper_2404_08970_b200 import api
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(3)

    def prob(n, m):
        x, y = np.sort(rng.random(n)), np.sort(rng.random(m))
        p, q = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
        return x, y, p, q

    # gradients: k = 1 (tiles + tails), k = 2, k = 3
    n, m = 300, 517
    x, y, p, q = prob(n, m)
    T = api.plan_buffer(n, m, dev)
    T.copy_(torch.rand(n, m, device=dev) / (n * m))
    for k in (1, 2, 3):
        api.grad(x, y, p, q, T, k=k)
    # solver: cluster-resident small path, then the multi-kernel fused / safe route, FGW, tau != eps
    x, y, p, q = prob(200, 150)
    api.solve(x, y, p, q, 0.02, 2, 20, device=dev, trace_objective=True)
    os.environ["GWDP_NO_SMALL"] = "1"
    api.solve(x, y, p, q, 0.02, 2, 20, device=dev, trace_objective=True)
    api.solve(x, y, p, q, 0.02, 2, 20, device=dev, fx=rng.random(200), fy=rng.random(150), alpha=0.5)
    api.solve(x, y, p, q, 0.02, 2, 20, device=dev, tau=0.01)
    api.solve(x, y, p, q, 0.02, 2, 10, device=dev, tol=1e-7, check_every=5)
    # fused path with a multi-CTA cluster spanning a row (m > 8192) and a ragged last CTA
    x2, y2, p2, q2 = prob(40, 9001)
    api.solve(x2, y2, p2, q2, 0.05, 1, 6, device=dev)
    os.environ.pop("GWDP_NO_SMALL")
    api.solve(x, y, p, q, 0.02, 2, 20, device=dev, k=3)
    # 2-D grids, unbalanced GW
    s = np.arange(9) / 8.0
    u = rng.dirichlet(np.ones(81))
    api.solve(s, s, u, u[::-1].copy(), 0.02, 2, 20, device=dev, grid2d=True, trace_objective=True)
    api.ugw_solve(x, y, p, q, 1.0, 0.02, 2, 10, device=dev, trace_objective=True)
    torch.cuda.synchronize()
    # fp64 storage (GW_F64, f64.cuh): gradient (in place and with supplied moments), Sinkhorn with the
    # tolerance rule, a graph-captured solve with the objective trace, FGW
    n, m = 133, 70
    x, y, p, q = prob(n, m)
    T64 = api.plan_buffer(n, m, dev, torch.float64)
    T64.copy_(torch.from_numpy(rng.random((n, m)) / (n * m)))
    Tn = T64.cpu().numpy()
    api.grad(x, y, p, q, T64, moments=(Tn.sum(1), Tn @ y, Tn.sum(0), Tn.T @ x))
    api.grad(x, y, p, q, T64, out=T64)
    api.sinkhorn(T64, p, q, 0.05, 25, tol=1e-12, check_every=5, return_plan=True)
    api.solve(x, y, p, q, 0.02, 2, 20, device=dev, trace_objective=True, return_plan=True, dtype=torch.float64)
    api.solve(x, y, p, q, 0.02, 2, 20, device=dev, fx=rng.random(n), fy=rng.random(m), alpha=0.5,
              dtype=torch.float64)
    torch.cuda.synchronize()
    print("sanitize workload ok")


if __name__ == "__main__":
    main()
