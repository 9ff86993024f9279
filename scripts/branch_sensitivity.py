#!/usr/bin/env python
"""Trajectory-sensitivity diagnostic for solve cases whose GPU objective deviates from the float64 oracle
(reading R25).  Runs the oracle's own mirror-descent iteration (built from
oracle.grad_prescribed / sinkhorn / plan_from_duals / objective) on the case's inputs

  * in float64 (the parity oracle),
  * with every subproblem's cost rounded to fp32 (the storage BASELINE.json prescribes),
  * with the fp32 cost perturbed by +-u ulp at random per entry (ensembles of seeds: rounding-level noise
    of the size an fp32-storage / fp32-exponent implementation makes),

and prints E(T^l) per outer iteration for each, so a deviation can be attributed to the amplification of
rounding-level differences by the iteration itself (the spread of the ensemble) rather than to an error.

    python scripts/branch_sensitivity.py gpurun_out/fail_206.npz [--outer 3 --inner 60 --seeds 8]
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle as O  # noqa: E402


def trajectory(x, y, p, q, eps, outer, inner, k, cost=None):
    T = np.outer(p, q)
    f = np.zeros(x.size)
    g = np.zeros(y.size)
    E = []
    for l in range(outer):
        G = O.grad_prescribed(x, y, p, q, T, k)
        if cost is not None:
            G = cost(G, l)
        f, g, _ = O.sinkhorn(G, p, q, eps, inner, f, g)
        T = O.plan_from_duals(G, f, g, eps)
        E.append(O.objective(x, y, T, k))
    return E


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("case")
    ap.add_argument("--outer", type=int, default=3)
    ap.add_argument("--inner", type=int, default=60)
    ap.add_argument("--seeds", type=int, default=8)
    ap.add_argument("--ulps", type=int, nargs="+", default=[1, 8],
                    help="perturbation sizes (fp32 ulps of the cost) of the noise ensembles")
    args = ap.parse_args()
    d = np.load(args.case)
    x, y, p, q, eps, k = d["x"], d["y"], d["p"], d["q"], float(d["eps"]), int(d["k"])
    E64 = trajectory(x, y, p, q, eps, args.outer, args.inner, k)
    E32 = trajectory(x, y, p, q, eps, args.outer, args.inner, k,
                     cost=lambda G, l: G.astype(np.float32).astype(np.float64))
    rel = lambda a: [abs(ai - bi) / abs(bi) for ai, bi in zip(a, E64)]  # noqa: E731
    out = {"case": os.path.basename(args.case), "n": int(x.size), "m": int(y.size), "eps": eps, "k": k,
           "outer": args.outer, "inner": args.inner,
           "E_fp64": E64, "E_fp32_cost": E32, "rel_fp32_cost_vs_fp64": rel(E32)}
    for u in args.ulps:
        ens = []
        for s_ in range(args.seeds):
            rng = np.random.default_rng(s_)

            def noisy(G, l, rng=rng):
                G32 = G.astype(np.float32)
                # +-u ulp at random per entry: u steps of nextafter towards +inf or -inf
                step = rng.choice([-1, 1], size=G.shape)
                ulp = np.spacing(np.abs(G32)).astype(np.float64)
                return G32.astype(np.float64) + step * u * ulp
            ens.append(trajectory(x, y, p, q, eps, args.outer, args.inner, k, cost=noisy))
        ens = np.asarray(ens)
        out["ensemble_%dulp_rel_spread" % u] = [float((ens[:, l].max() - ens[:, l].min()) / abs(E64[l]))
                                               for l in range(args.outer)]
        out["ensemble_%dulp_max_rel_dev_vs_fp64" % u] = [float(np.max(np.abs(ens[:, l] - E64[l])) / abs(E64[l]))
                                                        for l in range(args.outer)]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
