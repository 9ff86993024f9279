#!/usr/bin/env python
"""Timing of the GW_F64 storage path (f64.cuh): one JSON line per case, device-timed
with CUDA events on the library stream after warm-up; inputs seeded and synthetic (workloads/).

    python scripts/bench_f64.py > profiles/r02_f64_timing.jsonl

Cases: the C1 solve (BASELINE configs[0], 256 x 256, 20 x 100) with fp64 and with fp32 storage; the fp64
gradient and one fp64 Sinkhorn iteration at 4096^2 and 16384^2 against MEASURED_PEAKS.json hbm_gbs, with
algorithmic bytes 16 N M per gradient (read T, write G) and 8 N M per iteration (one read of G), and the
bytes this design moves (40 N M: T read, B write, B read twice, G write; 16 N M: a row and a column read).
"""

import json
import os
import sys

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


def main():
    import numpy as np
    import torch
    import __graft_entry__ as ge
    ge.build()
    import workloads as W
    from paper_2404_08970_b200 import api
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream(dev)
    peak = hbm_peak()
    P = W.config1()
    for dt in (torch.float64, torch.float32):
        api.solve(P.x, P.y, P.p, P.q, P.eps, P.outer, P.inner, dtype=dt)
        ms = [api.solve(P.x, P.y, P.p, P.q, P.eps, P.outer, P.inner, dtype=dt).ms_total for _ in range(5)]
        print(json.dumps({"case": "C1 solve 256x256, 20 x 100", "storage": str(dt).split(".")[-1],
                          "ms_total_median": float(np.median(ms)), "outer_it_per_s": P.outer / (np.median(ms) / 1e3)}),
              flush=True)
    for n in (4096, 16384):
        rng = np.random.default_rng(n)
        x, y = np.sort(rng.random(n)), np.sort(rng.random(n))
        p = q = np.full(n, 1.0 / n)
        T = api.plan_buffer(n, n, dev, torch.float64)
        T.copy_(torch.from_numpy(rng.exponential(size=(n, n)) / (n * n)))
        G = api.plan_buffer(n, n, dev, torch.float64)
        ms = timed(lambda: api.grad(x, y, p, q, T, out=G), 5, st)
        nm = float(n) * n
        print(json.dumps({"case": "fp64 gradient", "n": n, "m": n, "ms": ms,
                          "algorithmic_GBps": 16 * nm / ms / 1e6, "frac_algorithmic": 16 * nm / ms / 1e6 / peak,
                          "design_GBps": 40 * nm / ms / 1e6, "frac_design": 40 * nm / ms / 1e6 / peak,
                          "peak_GBps": peak}), flush=True)
        it = 20
        ms = timed(lambda: api.sinkhorn(G, p, q, 0.05, it), 2, st) / it
        print(json.dumps({"case": "fp64 Sinkhorn iteration", "n": n, "m": n, "ms": ms,
                          "algorithmic_GBps": 8 * nm / ms / 1e6, "frac_algorithmic": 8 * nm / ms / 1e6 / peak,
                          "design_GBps": 16 * nm / ms / 1e6, "frac_design": 16 * nm / ms / 1e6 / peak}), flush=True)
        del T, G
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
