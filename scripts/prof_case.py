#!/usr/bin/env python
"""Small driver for ncu captures of one kernel family (one case per run, sizes chosen so that ncu's
replays stay short; HBM-bound behaviour is the same as at C4):

  gibbs   entropic_gw_solve, N = M = 16384, 2 outer x 5 inner: the second gradient runs the solver's
          Gibbs-mode kernels (k_grad_moments3<1>, k_grad_store2<1,...>)
  k3      gw_grad_dp, k = 3, explicit plan, N = M = 16384 (k_gk_sums / k_gk_main)
  k4      as k3 with k = 4
  grid2d  gw_grad_dp GW_GRID2D, 128 x 128 grids (N = M = 16384) (k_g2_rowred / k_g2_store)

    python scripts/prof_case.py gibbs
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    case = sys.argv[1]
    import numpy as np
    import torch
    import workloads as W
    from paper_2404_08970_b200 import api
    dev = torch.device("cuda", 0)
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
    rng = np.random.default_rng(0)
    if case == "gibbs":
        P = W.config4(n)
        api.solve(P.x, P.y, P.p, P.q, P.eps, 2, 5, device=dev)
    elif case in ("k3", "k4", "k3big", "k5big"):
        k = int(case[1])
        if case.endswith("big"):
            n = 65536
        x = np.sort(rng.random(n))
        p = np.full(n, 1.0 / n)
        T = api.plan_buffer(n, n, dev)
        T.copy_(torch.rand((n, n), device=dev) / (n * n))
        G = torch.empty_like(T)
        for _ in range(2):
            api.grad(x, x, p, p, T, out=G, k=k)
    elif case in ("grid2d", "grid2d256"):
        side = 128 if case == "grid2d" else 256
        s = np.arange(side) / (side - 1.0)
        w = rng.random(side * side) + 0.05
        w /= w.sum()
        T = api.plan_buffer(side * side, side * side, dev)
        T.copy_(torch.rand((side * side, side * side), device=dev) / (side ** 4))
        G = torch.empty_like(T)
        api.grad(s, s, w, w, T, out=G, grid2d=True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            api.grad(s, s, w, w, T, out=G, grid2d=True)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        nm = float(side) ** 4
        print("grid2d %dx%d gradient %.3f ms, %.0f GB/s over 8NM" % (side, side, ms, 8 * nm / ms / 1e6))
    elif case == "ugw":
        # UGW at 16384^2 (rho = 1, eps = 1e-2, 2 outer x 50 inner): graph path vs instrumented breakdown
        import ctypes as C
        from paper_2404_08970_b200 import _lib
        x3, y3 = np.sort(rng.random(n)), np.sort(rng.random(n))
        u3 = rng.random(n) + 0.5
        u3 /= u3.sum()
        v3 = rng.random(n) + 0.5
        v3 *= 1.3 / v3.sum()
        ctx = api.Context.get(dev)
        api.ugw_solve(x3, y3, u3, v3, 1.0, 1e-2, 2, 50, device=dev)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = api.ugw_solve(x3, y3, u3, v3, 1.0, 1e-2, 2, 50, device=dev)
        e1.record()
        torch.cuda.synchronize()
        print("ugw graph path: %.3f ms, fused %d" % (e0.elapsed_time(e1), r.inner_fused_total))
        lib = _lib.load()
        ms_c = (C.c_double * 8)()
        cnt_c = (C.c_int64 * 8)()
        _lib.check(lib.gw_ctx_profile(ctx.h, 2, None, None, 0))
        e0.record()
        api.ugw_solve(x3, y3, u3, v3, 1.0, 1e-2, 2, 50, device=dev)
        e1.record()
        torch.cuda.synchronize()
        _lib.check(lib.gw_ctx_profile(ctx.h, 0, C.cast(ms_c, C.c_void_p), C.cast(cnt_c, C.c_void_p), 8))
        names = ["grad_moments", "grad_carry", "grad_main", "sink_row", "sink_col", "sink_fused", "objective"]
        print("ugw instrumented: %.3f ms; classes: %s" % (e0.elapsed_time(e1),
              {nm: round(ms_c[i], 3) for i, nm in enumerate(names)}))
    elif case == "c3grad":
        # gw_grad_dp on an explicit plan at N = M = n (C3: 16384), per kernel class (instrumented) + plain
        import ctypes as C
        from paper_2404_08970_b200 import _lib
        x, y = np.sort(rng.random(n)), np.sort(rng.random(n))
        p = np.full(n, 1.0 / n)
        T = api.plan_buffer(n, n, dev)
        T.copy_(torch.rand((n, n), device=dev) / (n * n))
        ctx = api.Context.get(dev)
        lib = _lib.load()
        for _ in range(3):
            api.grad(x, y, p, p, T)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            api.grad(x, y, p, p, T)
        e1.record()
        torch.cuda.synchronize()
        print("gw_grad_dp %d^2: %.4f ms per call" % (n, e0.elapsed_time(e1) / 10))
        ms_c = (C.c_double * 10)()
        cnt_c = (C.c_int64 * 10)()
        _lib.check(lib.gw_ctx_profile(ctx.h, 2, None, None, 0))
        for _ in range(10):
            api.grad(x, y, p, p, T)
        _lib.check(lib.gw_ctx_profile(ctx.h, 0, C.cast(ms_c, C.c_void_p), C.cast(cnt_c, C.c_void_p), 10))
        print({nm: round(ms_c[i] / 10, 4) for i, nm in enumerate(["moments", "carry", "main"])})
    elif case == "onepass":
        # the solver's gradient on the one-read path (rowclu.cuh) and the XM sweep that feeds it, C4 recipe
        # at N = M = n: 3 outer x 3 inner, instrumented (eager launches); then the two-read path
        import ctypes as C
        import os
        from paper_2404_08970_b200 import _lib
        import workloads as W
        P = W.config4(n)
        ctx = api.Context.get(dev)
        lib = _lib.load()
        names = ["grad_moments", "grad_carry", "grad_main", "sink_row", "sink_col", "sink_fused", "objective",
                 None, "grad_onepass", "sink_xm"]
        os.environ["GWDP_RC"] = "1"
        for env in ("", "1"):
            os.environ["GWDP_NO_RC"] = env
            api.solve(P.x, P.y, P.p, P.q, P.eps, 2, 3, device=dev)
            ms_c = (C.c_double * 10)()
            cnt_c = (C.c_int64 * 10)()
            _lib.check(lib.gw_ctx_profile(ctx.h, 2, None, None, 0))
            r = api.solve(P.x, P.y, P.p, P.q, P.eps, 4, 3, device=dev)
            _lib.check(lib.gw_ctx_profile(ctx.h, 0, C.cast(ms_c, C.c_void_p), C.cast(cnt_c, C.c_void_p), 10))
            print("GWDP_NO_RC=%s onepass=%d:" % (env or "0", r.grad_onepass_total),
                  {nm: (round(ms_c[i], 3), int(cnt_c[i])) for i, nm in enumerate(names) if nm and cnt_c[i]})
        os.environ.pop("GWDP_NO_RC", None)
    else:
        raise SystemExit("unknown case %s" % case)
    torch.cuda.synchronize()
    print("ok", case)


if __name__ == "__main__":
    main()
