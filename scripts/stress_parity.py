#!/usr/bin/env python
"""Randomised parity sweep (beyond the committed tests): many seeded random shapes, ties, marginals
and distance powers through the C ABI against the float64 oracle.

    python scripts/stress_parity.py [--cases 300] [--seed 0] [--f64]

Prints one line per failure and a summary; exit status 1 if any case fails.
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=300)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--dump", default=None, help="directory for the inputs of failing solve cases")
    ap.add_argument("--f64", action="store_true", help="also GW_F64 (fp64 storage) gradients and solves")
    args = ap.parse_args()
    import numpy as np
    import torch
    import oracle as O
    from paper_2404_08970_b200 import api
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(args.seed)
    fails = 0
    worst = {}
    devs = {}  # solve deviations per input class

    def note(kind, err, tol, info):
        nonlocal fails
        worst[kind] = max(worst.get(kind, 0.0), err / tol)
        if not err <= tol:
            fails += 1
            print("FAIL %s err %.3g tol %.3g %s" % (kind, err, tol, info), flush=True)

    def supports(n):
        x = np.sort(rng.random(n) * rng.choice([1.0, 10.0, 0.01]) + rng.normal())
        if n > 4 and rng.random() < 0.5:
            i = rng.integers(1, n)
            x[i] = x[i - 1]  # a tie
        return x

    def marg(n):
        w = rng.dirichlet(np.ones(n) * rng.choice([0.3, 1.0, 5.0]))
        if n > 3 and rng.random() < 0.2:
            w[rng.integers(0, n)] = 0.0  # a zero-mass point
            w /= w.sum()
        return w

    for case in range(args.cases):
        kind = rng.choice(["grad", "grad", "grad", "solve", "grid"] + (["grad64", "solve64"] if args.f64 else []))
        try:
            if kind == "grad":
                n, m = int(rng.integers(1, 1500)), int(rng.integers(1, 1500))
                k = int(rng.choice([1, 1, 2, 3, 4, 5]))
                x, y, p, q = supports(n), supports(m), marg(n), marg(m)
                T = (rng.random((n, m)) ** rng.choice([1, 3])).astype(np.float32)
                T /= T.sum()
                Td = api.plan_buffer(n, m, dev)
                Td.copy_(torch.from_numpy(T))
                G = api.grad(x, y, p, q, Td, k=k).cpu().numpy().astype(np.float64)
                Go = O.grad_prescribed(x, y, p, q, T.astype(np.float64), k=k)
                note("grad k=%d" % k, np.max(np.abs(G - Go)) / max(np.max(np.abs(Go)), 1e-300), 1e-5,
                     "n=%d m=%d" % (n, m))
            elif kind == "solve":
                n, m = int(rng.integers(2, 400)), int(rng.integers(2, 400))
                k = int(rng.choice([1, 1, 2, 3]))
                # both input classes: iid uniform supports (C1 / C4's recipe) and asymmetric Beta supports
                # (C5's); reading R25 -- near-symmetric instances can branch -- is checked, not assumed:
                # a deviating case is replayed by the oracle with the cost rounded to fp32 (the storage
                # BASELINE prescribes) to show whether the fp32 storage alone moves the trajectory there
                iid = rng.random() < 0.5
                if iid:
                    x, y = np.sort(rng.random(n)), np.sort(rng.random(m))
                else:
                    x, y = np.sort(rng.beta(2, 5, n)), np.sort(rng.beta(5, 2, m))
                p, q = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
                eps = float(rng.choice([0.01, 0.02, 0.05]))
                small = rng.random() < 0.5
                if not small:
                    os.environ["GWDP_NO_SMALL"] = "1"
                r = api.solve(x, y, p, q, eps, 3, 60, device=dev, k=k)
                os.environ.pop("GWDP_NO_SMALL", None)
                ro = O.entropic_gw(x, y, p, q, eps, 3, 60, k=k)
                E = ro["gw_objective"]
                err = abs(r.gw_objective - E) / abs(E)
                cls = "iid" if iid else "beta"
                devs.setdefault(cls, []).append(err)
                info = "case=%d %s n=%d m=%d eps=%g k=%d small=%s" % (case, cls, n, m, eps, k, small)
                if err > 1e-4:
                    # diagnostic: the same float64 iteration with the cost stored in fp32
                    r32 = O.entropic_gw(x, y, p, q, eps, 3, 60, k=k, cost_dtype=np.float32)
                    e32 = abs(r32["gw_objective"] - E) / abs(E)
                    g32 = abs(r.gw_objective - r32["gw_objective"]) / abs(r32["gw_objective"])
                    info += " | fp32-cost oracle vs fp64 oracle %.3g, GPU vs fp32-cost oracle %.3g" % (e32, g32)
                    if args.dump:
                        np.savez(os.path.join(args.dump, "fail_%d.npz" % case), x=x, y=y, p=p, q=q, eps=eps, k=k)
                note("solve k=%d" % k, err, 1e-4, info)
            elif kind == "grad64":  # fp64 storage: rounding-level parity
                n, m = int(rng.integers(1, 1500)), int(rng.integers(1, 1500))
                k = int(rng.choice([1, 1, 2, 3, 4, 5]))
                x, y, p, q = supports(n), supports(m), marg(n), marg(m)
                T = rng.random((n, m)) ** rng.choice([1, 3])
                T /= T.sum()
                Td = api.plan_buffer(n, m, dev, torch.float64)
                Td.copy_(torch.from_numpy(T))
                G = api.grad(x, y, p, q, Td, k=k).cpu().numpy()
                Go = O.grad_prescribed(x, y, p, q, T, k=k)
                note("grad64 k=%d" % k, np.max(np.abs(G - Go)) / max(np.max(np.abs(Go)), 1e-300), 1e-13,
                     "n=%d m=%d" % (n, m))
            elif kind == "solve64":
                n, m = int(rng.integers(2, 400)), int(rng.integers(2, 400))
                k = int(rng.choice([1, 1, 2, 3]))
                iid = rng.random() < 0.5
                if iid:
                    x, y = np.sort(rng.random(n)), np.sort(rng.random(m))
                else:
                    x, y = np.sort(rng.beta(2, 5, n)), np.sort(rng.beta(5, 2, m))
                p, q = rng.dirichlet(np.ones(n)), rng.dirichlet(np.ones(m))
                eps = float(rng.choice([0.01, 0.02, 0.05]))
                r = api.solve(x, y, p, q, eps, 3, 60, device=dev, k=k, dtype=torch.float64)
                ro = O.entropic_gw(x, y, p, q, eps, 3, 60, k=k)
                E = ro["gw_objective"]
                err = abs(r.gw_objective - E) / abs(E)
                cls = "f64 " + ("iid" if iid else "beta")
                devs.setdefault(cls, []).append(err)
                note("solve64 k=%d" % k, err, 1e-10, "case=%d %s n=%d m=%d eps=%g k=%d" % (case, cls, n, m, eps, k))
            else:
                nx, ny = int(rng.integers(1, 20)), int(rng.integers(1, 20))
                sx, sy = np.sort(rng.random(nx)), np.sort(rng.random(ny))
                p, q = marg(nx * nx), marg(ny * ny)
                T = rng.random((nx * nx, ny * ny)).astype(np.float32)
                T /= T.sum()
                Td = api.plan_buffer(nx * nx, ny * ny, dev)
                Td.copy_(torch.from_numpy(T))
                G = api.grad(sx, sy, p, q, Td, grid2d=True).cpu().numpy().astype(np.float64)
                Go = O.grad_prescribed_2d(sx, sy, p, q, T.astype(np.float64))
                note("grid2d", np.max(np.abs(G - Go)) / max(np.max(np.abs(Go)), 1e-300), 1e-5,
                     "nx=%d ny=%d" % (nx, ny))
        except Exception as e:  # noqa: BLE001 - report and continue
            fails += 1
            print("ERROR %s case %d: %r" % (kind, case, e), flush=True)
    print("stress: %d cases, %d failures; worst err/tol per kind: %s" % (
        args.cases, fails, {k: round(v, 3) for k, v in sorted(worst.items())}), flush=True)
    for cls, v in sorted(devs.items()):
        v = np.sort(np.asarray(v))
        print("solve deviation distribution (%s supports, %d cases): median %.2e, p90 %.2e, p99 %.2e, max %.2e; "
              "above 1e-4: %d" % (cls, v.size, np.median(v), np.quantile(v, 0.9), np.quantile(v, 0.99), v[-1],
                                  int(np.sum(v > 1e-4))), flush=True)
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
