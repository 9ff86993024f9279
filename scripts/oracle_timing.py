#!/usr/bin/env python
"""SURVEY §8(d) host-oracle timing protocol: the float64 NumPy oracle (oracle/) timed on the host cores
of the box it runs on (context for the GPU numbers, never a target).  One JSON line per measurement:

  * c3 (grad_prescribed: two dense DGEMMs) at N = 256, 4096, 16384 on C3's plan;
  * one c7 Sinkhorn iteration (oracle.sinkhorn) at the same sizes;
  * the full C1 solve (oracle.entropic_gw, 20 outer x 100 inner, N = 256);
  * c3 at N = 4096 with ONE BLAS thread -- the paper's own setting is a single thread on a Xeon Gold
    5117.

    python scripts/oracle_timing.py > profiles/r02_oracle_timing.jsonl
"""

import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
import workloads as W  # noqa: E402


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def blas_info():
    try:
        from threadpoolctl import threadpool_info
        return [{"api": d.get("internal_api"), "threads": d.get("num_threads")} for d in threadpool_info()]
    except Exception:
        return None


def timeit(fn, reps=1):
    fn()  # warm (allocations, BLAS thread pool)
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t0) / reps


def main():
    host = {"cores": len(os.sched_getaffinity(0)), "cpu": cpu_model(), "blas": blas_info(),
            "numpy": np.__version__}

    def emit(d):
        d["host"] = host
        print(json.dumps(d), flush=True)

    for n in (256, 4096, 16384):
        P = W.config3(n)
        T = P.extra["T"].astype(np.float64)
        reps = 5 if n <= 4096 else 1
        t = timeit(lambda: O.grad_prescribed(P.x, P.y, P.p, P.q, T), reps)
        emit({"what": "c3 grad_prescribed (dense, two DGEMMs)", "N": n, "M": n, "s": t, "threads": "all"})
        G = O.grad_prescribed(P.x, P.y, P.p, P.q, T)
        t = timeit(lambda: O.sinkhorn(G, P.p, P.q, 1e-3, 1), reps)
        emit({"what": "c7 one Sinkhorn iteration (f- then g-update, log-domain)", "N": n, "M": n, "s": t,
              "eps": 1e-3, "threads": "all"})
        del T, G
    C1 = W.config1()
    t = timeit(lambda: O.entropic_gw(C1.x, C1.y, C1.p, C1.q, C1.eps, C1.outer, C1.inner), 1)
    emit({"what": "c8 full C1 solve (20 outer x 100 inner)", "N": 256, "M": 256, "s": t, "threads": "all"})
    try:
        from threadpoolctl import threadpool_limits
        P = W.config3(4096)
        T = P.extra["T"].astype(np.float64)
        with threadpool_limits(limits=1):
            t = timeit(lambda: O.grad_prescribed(P.x, P.y, P.p, P.q, T), 2)
        emit({"what": "c3 grad_prescribed, ONE BLAS thread (the paper's single-thread setting, PAPER.md:409)",
              "N": 4096, "M": 4096, "s": t, "threads": 1})
    except ImportError:
        emit({"what": "c3 single-thread", "skipped": "threadpoolctl not importable"})


if __name__ == "__main__":
    main()
