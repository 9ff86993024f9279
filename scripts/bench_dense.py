#!/usr/bin/env python
"""the DP gradient against the dense product it replaces, on C3
(BASELINE configs[2]: N = M = 16384, T = Exp(1) rescaled to uniform marginals, x, y sorted U[0,1)).

    python scripts/bench_dense.py [--n 16384] > profiles/dense_compare_rNN.jsonl

The dense comparison point materialises D_X, D_Y and forms G = 2(c 1^T + 1 c'^T) - 4 D_X T D_Y
with cuBLAS (torch.matmul) in fp64, fp32, TF32 and bf16 (tensor cores for the last two).  Every
variant is timed with CUDA events (best of 3 after a warm-up) and its max-abs error is reported
against the fp64 dense result, which is itself checked against the float64 CPU oracle on sampled
rows.  One JSON line per variant.
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16384)
    args = ap.parse_args()
    import numpy as np
    import torch
    import oracle as O
    import workloads as W
    from paper_2404_08970_b200 import api
    dev = torch.device("cuda", 0)
    P = W.config3(args.n)
    n = args.n
    x = torch.tensor(P.x, dtype=torch.float64, device=dev)
    y = torch.tensor(P.y, dtype=torch.float64, device=dev)
    p = torch.tensor(P.p, dtype=torch.float64, device=dev)
    q = torch.tensor(P.q, dtype=torch.float64, device=dev)
    T32 = torch.from_numpy(np.ascontiguousarray(P.extra["T"], dtype=np.float32)).to(dev)
    del P.extra["T"]

    def timed(fn, reps=3):
        fn()
        torch.cuda.synchronize()
        best = float("inf")
        out = None
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            out = fn()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return best, out

    # fp64 dense reference on the GPU (D materialised, two DGEMMs)
    DX = (x[:, None] - x[None, :]).abs()
    DY = (y[:, None] - y[None, :]).abs()
    c1 = (DX * DX) @ p
    c2 = (DY * DY) @ q
    T64 = T32.double()
    ms64, Gref = timed(lambda: 2.0 * (c1[:, None] + c2[None, :]) - 4.0 * (DX @ T64 @ DY), reps=2)
    scale = Gref.abs().max().item()
    print("diag: Gref finite %s max %r c1 max %r T max %r sum %r" % (
        bool(torch.isfinite(Gref).all().item()), scale, c1.abs().max().item(), T32.max().item(),
        T32.double().sum().item()), file=sys.stderr, flush=True)
    # tie the GPU fp64 reference to the CPU oracle on sampled rows: rows of D_X T D_Y by a
    # float64 NumPy product of the sampled rows of D_X with T, then with D_Y
    rng = np.random.default_rng(0)
    rows = np.sort(rng.choice(n, 8, replace=False))
    Tn = T64.cpu().numpy()
    xs, ys = P.x, P.y
    DXr = np.abs(xs[rows][:, None] - xs[None, :])
    DYn = np.abs(ys[:, None] - ys[None, :])
    cr = O.const_term(xs, ys, P.p, P.q)
    Go_rows = 2.0 * (cr[0][rows][:, None] + cr[1][None, :]) - 4.0 * ((DXr @ Tn) @ DYn)
    ref_err = float(np.max(np.abs(Gref[rows].cpu().numpy() - Go_rows)) / scale)
    del Tn, DYn
    lines = [{"variant": "dense fp64 (cuBLAS DGEMM, D materialised)", "N": n, "ms": ms64,
              "max_abs_err_rel": 0.0, "vs_oracle_sampled_rows": ref_err}]
    flops = 2.0 * 2 * n ** 3
    lines[0]["TFLOPs"] = flops / ms64 / 1e9

    # DP gradient (this library)
    G = api.plan_buffer(n, n, dev)
    msdp, _ = timed(lambda: api.grad(x, y, p, q, T32, out=G, validate=False))
    err = ((G.double() - Gref).abs().max().item()) / scale
    lines.append({"variant": "DP gradient gw_grad_dp (fp32 data, fp64 carries)", "N": n, "ms": msdp,
                  "max_abs_err_rel": err, "GBps_12NM": 12.0 * n * n / msdp / 1e6})
    del G
    torch.cuda.empty_cache()

    def dense(dt, tf32):
        torch.backends.cuda.matmul.allow_tf32 = tf32
        DXd, DYd, Td = DX.to(dt), DY.to(dt), T32.to(dt)
        c1d, c2d = c1.to(torch.float32), c2.to(torch.float32)

        def run():
            V = (DXd @ Td) @ DYd
            return 2.0 * (c1d[:, None] + c2d[None, :]) - 4.0 * V.float()
        ms, Gd = timed(run)
        e = ((Gd.double() - Gref).abs().max().item()) / scale
        torch.backends.cuda.matmul.allow_tf32 = False
        return ms, e

    for name, dt, tf in [("dense fp32 (cuBLAS SGEMM, no TF32)", torch.float32, False),
                         ("dense TF32 tensor cores", torch.float32, True),
                         ("dense bf16 tensor cores (fp32 accumulate)", torch.bfloat16, False)]:
        ms, e = dense(dt, tf)
        lines.append({"variant": name, "N": n, "ms": ms, "max_abs_err_rel": e, "TFLOPs": flops / ms / 1e9,
                      "within_north_star_tol_1e-5": e <= 1e-5})
    for d in lines:
        d["speedup_of_DP"] = d["ms"] / msdp
        print(json.dumps(d), flush=True)


if __name__ == "__main__":
    main()
