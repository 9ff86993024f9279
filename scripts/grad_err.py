#!/usr/bin/env python
"""Max-abs error of the solver's own gradient G^l (exported, default two-read path) against the float64
oracle on the exported plan, for a few iid-uniform shapes; also the error in ulps of each entry.

    python scripts/grad_err.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    import oracle as O
    from paper_2404_08970_b200 import api
    dev = torch.device("cuda", 0)
    os.environ["GWDP_NO_SMALL"] = "1"
    for (n, m, eps, seed) in [(320, 375, 0.01, 75), (1000, 1000, 0.01, 1), (2048, 2048, 0.005, 2), (4096, 4096, 0.002, 3)]:
        rng = np.random.default_rng(seed)
        x, y = np.sort(rng.random(n)), np.sort(rng.random(m))
        p, q = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
        Tb, Gb = api.plan_buffer(n, m, dev), api.plan_buffer(n, m, dev)
        api.solve(x, y, p, q, eps, 3, 30, device=dev, export_iter=3, export_T=Tb, export_G=Gb)
        T = Tb.cpu().numpy().astype(np.float64)
        G = Gb.cpu().numpy().astype(np.float64)
        Go = O.grad_prescribed(x, y, p, q, T)
        err = np.abs(G - Go)
        ulp = np.spacing(np.abs(Go).astype(np.float32)).astype(np.float64)
        w = T / T.sum()
        print("n=%d m=%d eps=%g: max err / max|G| %.3e; err in ulps of the entry: median %.1f, p99 %.1f, "
              "plan-weighted mean %.2f" % (n, m, eps, err.max() / np.abs(Go).max(), np.median(err / ulp),
                                           np.percentile(err / ulp, 99), float((w * err / ulp).sum())))


if __name__ == "__main__":
    main()
