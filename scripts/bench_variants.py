#!/usr/bin/env python
"""Measurement of the SURVEY §8(f) rows built beside the hot path (FGW, k = 2..5, 2-D grids):
one JSON line per variant, device-timed with CUDA events on the library stream after warm-up.

    python scripts/bench_variants.py [--n 65536] [--reps 3] > profiles/variants_rNN.jsonl

Per variant: ms per unit, the unit's algorithmic bytes and the fraction of
MEASURED_PEAKS.json hbm_gbs; for the solves, outer iterations/s.  "oracle" times the float64
oracle on a small sample of the same recipe (context, not a target).  Inputs are synthetic and
seeded (workloads/); every matrix is larger than L2.
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def hbm_peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


def timed(fn, reps, stream):
    import torch
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def oracle_time(fn):
    t0 = time.perf_counter()
    fn()
    return time.perf_counter() - t0


SOLVE_BYTES_NOTE = ("2 outer iterations: gradient on T^0 = p q^T 4NM (write only) + gradient on the Gibbs plan "
                    "12NM + 4NM per one-read Sinkhorn iteration + the final objective 8NM")


def solve_bytes(inner, nm, outer=2, stats=0):
    """Algorithmic bytes of an `outer`-iteration solve with `inner` fused iterations per outer iteration
    (NM = N x M elements; 4NM = one fp32 pass over the matrix)."""
    return (4 + 12 * (outer - 1) + 4 * inner * outer + stats * outer + 8) * nm


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=65536)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--no-oracle", action="store_true")
    ap.add_argument("--grads-only", action="store_true", help="only the explicit-plan gradients k = 1..5")
    args = ap.parse_args()
    import numpy as np
    import torch
    import workloads as W
    from paper_2404_08970_b200 import api
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    ctx = api.Context(dev, stream)
    peak = hbm_peak()
    n = args.n
    out = []

    def emit(d):
        d["peak_GBps"] = peak
        if "GBps" in d:
            d["frac"] = d["GBps"] / peak
        print(json.dumps(d), flush=True)
        out.append(d)

    # ---- gradients on an explicit plan, N = M = n (C3 recipe shape) ----
    rng = np.random.default_rng(0)
    x = np.sort(rng.random(n))
    p = np.full(n, 1.0 / n)
    with torch.cuda.stream(stream):
        T = torch.rand((n, n), device=dev, dtype=torch.float32) / (n * n)
        G = torch.empty_like(T)
    torch.cuda.synchronize()
    nm = float(n) * n
    for k, nbytes, note in [(1, 12, "moments read + main read + write (gap-weighted scans)"),
                            (2, 8, "moments read + write (polynomial moments)"),
                            (3, 12, "sums read + main read + write (power-sum scans)"),
                            (4, 8, "moments read + write (polynomial moments, fp64 per-row polynomial)"),
                            (5, 12, "as k = 3")]:
        with torch.cuda.stream(stream):
            ms = timed(lambda: api.grad(x, x, p, p, T, out=G, ctx=ctx, k=k), args.reps, stream)
        d = {"variant": "gw_grad_dp k=%d" % k, "row": "a1-a4" if k == 1 else "f2", "N": n, "M": n,
             "ms": ms, "algorithmic_bytes": nbytes * nm, "bytes_note": note, "GBps": nbytes * nm / ms / 1e6}
        if not args.no_oracle:
            import oracle as O
            ns = 1024
            xs = np.sort(rng.random(ns))
            ps = np.full(ns, 1.0 / ns)
            Ts = np.full((ns, ns), 1.0 / ns / ns)
            t = oracle_time(lambda: O.grad_prescribed(xs, xs, ps, ps, Ts, k))
            d["oracle"] = {"N": ns, "s": t, "note": "dense grad_prescribed (two float64 DGEMMs), host cores"}
        emit(d)
    del T, G
    torch.cuda.empty_cache()
    if args.grads_only:
        return

    # ---- 2-D grids: side 256 (N = M = 65536), Table-3 style weights ----
    side = int(round(n ** 0.5))
    if side * side == n and side <= 256:
        s = np.arange(side) / (side - 1.0)
        pw = rng.random(n) + 0.05
        pw /= pw.sum()
        with torch.cuda.stream(stream):
            T = torch.rand((n, n), device=dev, dtype=torch.float32) / (n * n)
            G = torch.empty_like(T)
            ms = timed(lambda: api.grad(s, s, pw, pw, T, out=G, ctx=ctx, grid2d=True), args.reps, stream)
        d = {"variant": "gw_grad_dp GW_GRID2D", "row": "f3", "grid": "%dx%d" % (side, side), "N": n, "M": n,
             "ms": ms, "algorithmic_bytes": 8 * nm, "bytes_note": "reduction read + write", "GBps": 8 * nm / ms / 1e6}
        if not args.no_oracle:
            import oracle as O
            ss = np.arange(24) / 23.0
            ps = np.full(576, 1.0 / 576)
            t = oracle_time(lambda: O.grad_prescribed_2d(ss, ss, ps, ps, np.outer(ps, ps)))
            d["oracle"] = {"grid": "24x24", "s": t, "note": "dense grad_prescribed_2d"}
        emit(d)
        del T, G
        torch.cuda.empty_cache()
        # solve on the grid at the paper's 2-D eps (0.004)
        with torch.cuda.stream(stream):
            r = None

            def run2d():
                nonlocal r
                r = api.solve(s, s, pw, pw, 0.004, 2, 100, device=dev, ctx=ctx, grid2d=True)
            ms = timed(run2d, 1, stream)
        emit({"variant": "entropic_gw_solve GW_GRID2D", "row": "f3", "grid": "%dx%d" % (side, side), "eps": 0.004,
              "outer": 2, "inner": 100, "ms": ms, "outer_iter_per_s": 2 / (ms / 1e3),
              "inner_fused": r.inner_fused_total, "gw_objective": r.gw_objective,
              "marginal_violation": r.marginal_violation})
        torch.cuda.empty_cache()

    # ---- FGW on the C5 recipe at full size (N = 32768, M = 24576) ----
    P = W.config5()
    with torch.cuda.stream(stream):
        r = None

        def runf():
            nonlocal r
            r = api.solve(P.x, P.y, P.p, P.q, P.eps, 2, 100, fx=P.fx, fy=P.fy, alpha=0.5, device=dev, ctx=ctx)
        ms = timed(runf, 1, stream)
    nm5 = float(P.n) * P.m
    emit({"variant": "fgw_solve (C5)", "row": "f1", "N": P.n, "M": P.m, "alpha": 0.5, "eps": P.eps, "outer": 2,
          "inner": 100, "ms": ms, "outer_iter_per_s": 2 / (ms / 1e3), "inner_fused": r.inner_fused_total,
          "algorithmic_bytes": solve_bytes(100, nm5), "bytes_note": SOLVE_BYTES_NOTE,
          "GBps": solve_bytes(100, nm5) / ms / 1e6, "gw_objective": r.gw_objective,
          "marginal_violation": r.marginal_violation})
    # ---- k = 3 solve at C3 size ----
    n3 = 16384
    x3, y3 = np.sort(rng.random(n3)), np.sort(rng.random(n3))
    p3 = np.full(n3, 1.0 / n3)
    with torch.cuda.stream(stream):
        r = None

        def run3():
            nonlocal r
            r = api.solve(x3, y3, p3, p3, 1e-2, 2, 100, device=dev, ctx=ctx, k=3)
        ms = timed(run3, 1, stream)
    nm3 = float(n3) * n3
    emit({"variant": "entropic_gw_solve k=3", "row": "f2", "N": n3, "M": n3, "eps": 1e-2, "outer": 2,
          "inner": 100, "ms": ms, "outer_iter_per_s": 2 / (ms / 1e3), "inner_fused": r.inner_fused_total,
          "algorithmic_bytes": solve_bytes(100, nm3), "bytes_note": SOLVE_BYTES_NOTE,
          "GBps": solve_bytes(100, nm3) / ms / 1e6, "gw_objective": r.gw_objective})
    # ---- unbalanced GW (row f4) at N = M = 16384, rho = 1, eps = 1e-2 (readings R32-R35) ----
    u3 = rng.random(n3) + 0.5
    u3 /= u3.sum()
    v3 = rng.random(n3) + 0.5
    v3 *= 1.3 / v3.sum()
    with torch.cuda.stream(stream):
        r = None

        def runu():
            nonlocal r
            r = api.ugw_solve(x3, y3, u3, v3, 1.0, 1e-2, 2, 50, device=dev, ctx=ctx)
        ms = timed(runu, 1, stream)
    emit({"variant": "ugw_solve", "row": "f4", "N": n3, "M": n3, "rho": 1.0, "eps": 1e-2, "outer": 2,
          "inner": 50, "ms": ms, "outer_iter_per_s": 2 / (ms / 1e3), "inner_fused": r.inner_fused_total,
          "algorithmic_bytes": solve_bytes(50, nm3, stats=4),
          "bytes_note": SOLVE_BYTES_NOTE + "; plan statistics 4NM per outer (one read of the cost)",
          "GBps": solve_bytes(50, nm3, stats=4) / ms / 1e6})
    # ---- unbalanced GW on the C5 recipe at full size (N = 32768, M = 24576, rho = 1.0, BASELINE configs[4]) ----
    with torch.cuda.stream(stream):
        r = None

        def runu5():
            nonlocal r
            r = api.ugw_solve(P.x, P.y, P.p, P.q, 1.0, P.eps, 2, 100, device=dev, ctx=ctx)
        ms = timed(runu5, 1, stream)
    emit({"variant": "ugw_solve (C5)", "row": "f4", "N": P.n, "M": P.m, "rho": 1.0, "eps": P.eps, "outer": 2,
          "inner": 100, "ms": ms, "outer_iter_per_s": 2 / (ms / 1e3), "inner_fused": r.inner_fused_total,
          "algorithmic_bytes": solve_bytes(100, nm5, stats=4),
          "bytes_note": SOLVE_BYTES_NOTE + "; plan statistics 4NM per outer (one read of the cost)",
          "GBps": solve_bytes(100, nm5, stats=4) / ms / 1e6, "gw_objective": r.gw_objective})
    torch.cuda.empty_cache()
    # ---- tau != eps (reading R6) on the same problem: cost G + (eps - tau) ln T ----
    with torch.cuda.stream(stream):
        r = None

        def runt():
            nonlocal r
            r = api.solve(x3, y3, p3, p3, 1e-2, 2, 100, device=dev, ctx=ctx, tau=5e-3)
        ms = timed(runt, 1, stream)
    emit({"variant": "entropic_gw_solve tau=eps/2", "row": "a (tau)", "N": n3, "M": n3, "eps": 1e-2, "tau": 5e-3,
          "outer": 2, "inner": 100, "ms": ms, "outer_iter_per_s": 2 / (ms / 1e3), "inner_fused": r.inner_fused_total,
          "algorithmic_bytes": solve_bytes(100, nm3), "bytes_note": SOLVE_BYTES_NOTE,
          "GBps": solve_bytes(100, nm3) / ms / 1e6, "gw_objective": r.gw_objective})
    ctx.close()


if __name__ == "__main__":
    main()
