#!/usr/bin/env python
"""One fp64 gradient and two fp64 Sinkhorn iterations at N = M = 16384 (GW_F64) for an ncu capture:
    ncu --set full -k regex:k64_ python scripts/prof_f64.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch
    from paper_2404_08970_b200 import api
    n = 16384
    rng = np.random.default_rng(n)
    x, y = np.sort(rng.random(n)), np.sort(rng.random(n))
    p = q = np.full(n, 1.0 / n)
    dev = torch.device("cuda", 0)
    T = api.plan_buffer(n, n, dev, torch.float64)
    T.copy_(torch.from_numpy(rng.exponential(size=(n, n)) / (n * n)))
    G = api.grad(x, y, p, q, T)
    api.sinkhorn(G, p, q, 0.05, 2)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
