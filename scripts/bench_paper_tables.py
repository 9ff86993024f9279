#!/usr/bin/env python
"""The paper's own timing workloads (context only, never a target: the paper
timed a single-threaded C++ program on a Xeon Gold 5117).

    python scripts/bench_paper_tables.py > profiles/paper_tables_rNN.jsonl

Table 2: 1-D uniform grid x_i = y_i = (i-1)/(N-1), weights U[0,1] normalised,
k = 1, 10 mirror-descent iterations, eps = 0.002; GW and FGW (theta = 0.5, c_ip = |i - p| in index
units, i.e. features fx_i = i, fy_p = p).  Table 3: 2-D n x n grid on
[0,1]^2 (GW_GRID2D), eps = 0.004.  The paper does not state its inner Sinkhorn count; the runs use
reading R8's tolerance rule (violation <= 1e-7 checked every 10 iterations, cap 2000) and report
the inner iterations used.  Synthetic seeded weights (numpy default_rng(seed)); wall time of one
api.solve call (synchronised), median of 3 after a warm-up.
"""

import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

PAPER_T2 = {"GW": {500: 0.497, 1000: 2.13, 2000: 10.1, 4000: 50.1},
            "FGW": {500: 0.600, 1000: 2.54, 2000: 12.0, 4000: 57.3}}
PAPER_T3 = {"GW": {30: 1.73, 60: 55.3, 90: 301.0, 120: 965.0}}


def main():
    import numpy as np
    import torch
    from paper_2404_08970_b200 import api
    dev = torch.device("cuda", 0)

    def run(fn):
        fn()
        torch.cuda.synchronize()
        ts, r = [], None
        for _ in range(3):
            t0 = time.perf_counter()
            r = fn()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        return statistics.median(ts), r

    # FGW feature cost: c_ip = |i - p| in index units (R23, as the caption prints it) -- then
    # (1 - theta) c^2 reaches 8e6 >> eps and the subproblems do not converge within the cap: those rows
    # are labelled converged = false and are NOT comparable with the paper's converged times; and the
    # same cost on the unit interval (fx_i = (i - 1)/(N - 1), like the supports), which converges.
    variants = [("GW", None), ("FGW", "index"), ("FGW", "unit")]
    for metric, feat in variants:
        for N, tp in PAPER_T2[metric].items():
            rng = np.random.default_rng(N)
            x = np.arange(N) / (N - 1.0)
            u, v = rng.random(N), rng.random(N)
            u, v = u / u.sum(), v / v.sum()
            kw = {}
            if feat == "index":
                kw = dict(fx=np.arange(N, dtype=np.float64), fy=np.arange(N, dtype=np.float64), alpha=0.5)
            elif feat == "unit":
                kw = dict(fx=x.copy(), fy=x.copy(), alpha=0.5)
            t, r = run(lambda: api.solve(x, x, u, v, 0.002, 10, 2000, tol=1e-7, check_every=10, device=dev, **kw))
            row = {"table": "PAPER Table 2 (1-D)", "metric": metric, "N": N, "eps": 0.002, "outer": 10,
                   "gpu_solve_s": t, "paper_fgc_s": tp, "paper_hardware": "1 thread, Xeon Gold 5117",
                   "inner_iters_total": r.inner_iters_total, "converged": bool(r.converged),
                   "gw_objective": r.gw_objective, "marginal_violation": r.marginal_violation}
            if feat:
                row["feature_cost"] = ("c_ip = |i - p| in index units (R23): (1-theta) c^2 up to %.1e >> eps"
                                       % (0.5 * (N - 1) ** 2) if feat == "index" else
                                       "c_ip = |i - p| / (N - 1) (features on the unit interval, like the supports)")
            if not r.converged:
                row["note"] = ("NOT converged within the 2000-iteration cap of every outer iteration: not comparable "
                               "with the paper's (converged) time")
            print(json.dumps(row), flush=True)
    for n, tp in PAPER_T3["GW"].items():
        rng = np.random.default_rng(n)
        s = np.arange(n) / (n - 1.0)
        u, v = rng.random(n * n), rng.random(n * n)
        u, v = u / u.sum(), v / v.sum()
        t, r = run(lambda: api.solve(s, s, u, v, 0.004, 10, 2000, tol=1e-7, check_every=10, device=dev,
                                     grid2d=True))
        print(json.dumps({"table": "PAPER Table 3 (2-D)", "metric": "GW", "grid": "%dx%d" % (n, n), "N": n * n,
                          "eps": 0.004, "outer": 10, "gpu_solve_s": t, "paper_fgc_s": tp,
                          "paper_hardware": "1 thread, Xeon Gold 5117", "inner_iters_total": r.inner_iters_total,
                          "gw_objective": r.gw_objective, "marginal_violation": r.marginal_violation}), flush=True)


if __name__ == "__main__":
    main()
