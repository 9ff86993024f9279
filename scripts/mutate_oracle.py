#!/usr/bin/env python
"""Mutation check of the oracle's pins (task ③: "a plausible mistake anywhere in it -- a dropped
term, a wrong sign or index, a transposed operand -- fails one of them").

For every mutation below a copy of oracle/ + tests/ + workloads/ is made under a temporary
directory, ONE textual edit is applied to the copy of the oracle, and the CPU pin tests
(tests/test_oracle_pins.py, tests/test_oracle_ugw.py) run against it.  A mutation "survives" if the
pins still pass: that function is then unpinned.  Calls nothing but oracle/ and its tests.

    python scripts/mutate_oracle.py [--jobs 8] > profiles/r02_oracle_mutations.log
"""

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (file, function it sits in, old text, new text, what the mistake is)
MUTATIONS = [
    ("gw.py", "dist", "np.abs(x[:, None] - x[None, :]) ** k", "np.abs(x[:, None] - x[None, :]) ** (k + 1)", "wrong power"),
    ("gw.py", "const_term", "return (DX * DX) @ _f64(p), (DY * DY) @ _f64(q)", "return DX @ _f64(p), (DY * DY) @ _f64(q)", "c without the square"),
    ("gw.py", "const_term", "return (DX * DX) @ _f64(p), (DY * DY) @ _f64(q)", "return (DX * DX) @ _f64(p), (DY * DY) @ np.ones_like(_f64(q)) / len(q)", "c' with uniform weights"),
    # (relabelling the summed indices of grad_entrywise / objective_bruteforce is an EQUIVALENT mutant:
    # D_X and D_Y are symmetric, so "ijpq,jp->iq" computes the same matrix)
    ("gw.py", "grad_entrywise", 'np.einsum("ijpq,jq->ip", diff * diff, T)', 'np.einsum("ijpq,jq->ip", np.abs(diff), T)', "dropped square"),
    ("gw.py", "grad_entrywise", "diff = DX[:, :, None, None] - DY[None, None, :, :]\n    return 2.0", "diff = DX[:, :, None, None] + DY[None, None, :, :]\n    return 2.0", "sign inside the square"),
    ("gw.py", "grad_entrywise", "return 2.0 * np.einsum", "return 1.0 * np.einsum", "dropped factor 2"),
    ("gw.py", "triple_product_dense", "return dist(x, k) @ _f64(T) @ dist(y, k)", "return dist(x, k) @ _f64(T) @ dist(y, 1)", "D_Y at the wrong power"),
    ("gw.py", "grad_prescribed", "- 4.0 * triple_product_dense(x, y, T, k)", "- 2.0 * triple_product_dense(x, y, T, k)", "wrong factor on the product"),
    ("gw.py", "grad_prescribed", "return 2.0 * (c[:, None] + c2[None, :]) - 4.0 * triple_product_dense", "return 2.0 * (c[:, None] - c2[None, :]) - 4.0 * triple_product_dense", "sign of c'"),
    ("gw.py", "grad_prescribed_dp", "c2 = ref_dp_distance(_f64(q), _f64(y), 2 * k)", "c2 = ref_dp_distance(_f64(q), _f64(y), k)", "c' at power k"),
    ("gw.py", "grad_realized", "return grad_prescribed(x, y, T.sum(axis=1), T.sum(axis=0), T, k)", "return grad_prescribed(x, y, T.sum(axis=1), T.sum(axis=1), T, k)", "b from the row sums"),
    ("gw.py", "ref_dp_lower", "acc = acc + math.comb(r - 1, t - 1) * delta ** (r - t) * term", "acc = acc + math.comb(r - 1, t - 1) * delta ** (r - t + 1) * term", "gap exponent off by one"),
    ("gw.py", "ref_dp_lower", "acc = acc + math.comb(r - 1, t - 1) * delta", "acc = acc + math.comb(r, t - 1) * delta", "wrong binomial"),
    ("gw.py", "ref_dp_lower", "term = a[..., i, t - 1] + (v[..., i] if t == 1 else 0.0)", "term = a[..., i, t - 1] + (v[..., i] if t == r else 0.0)", "v added to the wrong order"),
    ("gw.py", "ref_dp_upper", "return ref_dp_lower(v[..., ::-1], -s[::-1], k)[..., ::-1].copy()", "return ref_dp_lower(v[..., ::-1], -s[::-1], k).copy()", "result not reversed back"),
    ("gw.py", "ref_dp_distance", "return ref_dp_lower(v, s, k) + ref_dp_upper(v, s, k)", "return ref_dp_lower(v, s, k) - ref_dp_upper(v, s, k)", "sign of the upper part"),
    ("gw.py", "triple_product_dp", "return ref_dp_distance(W.T, x, k).T", "return ref_dp_distance(W.T, x, 1).T", "left factor at k = 1"),
    ("gw.py", "objective_bruteforce", 'np.einsum("ijpq,ip,jq->", diff * diff, T, T)', 'np.einsum("ijpq,ip,jq->", np.abs(diff), T, T)', "dropped square"),
    ("gw.py", "objective_bruteforce", 'np.einsum("ijpq,ip,jq->", diff * diff, T, T)', 'np.einsum("ijpq,ij,pq->", diff * diff, T[:, :T.shape[0]] if T.shape[1] >= T.shape[0] else T, T[:T.shape[1], :] if T.shape[0] >= T.shape[1] else T)', "plan indexed by the wrong pair"),
    ("gw.py", "objective", "- 2.0 * np.sum((DX @ T @ DY) * T))", "- 1.0 * np.sum((DX @ T @ DY) * T))", "cross term factor"),
    ("gw.py", "objective", "return float(a @ (DX * DX) @ a + b @ (DY * DY) @ b", "return float(a @ (DX * DX) @ a + a @ (DX * DX) @ a", "b term replaced"),
    ("gw.py", "entropy", "(np.log(T[pos]) - 1.0)", "(np.log(T[pos]))", "dropped the -1"),
    ("gw.py", "violation", "np.max(np.abs(T.sum(axis=0) - _f64(q)))))", "np.max(np.abs(T.sum(axis=1) - _f64(p)))))", "rows only"),
    ("gw.py", "violation", "return float(max(np.max(np.abs(T.sum(axis=1) - _f64(p))),", "return float(max(np.max(np.abs(T.sum(axis=0) - _f64(q))),", "columns only"),
    ("gw.py", "fgw_grad_prescribed", "return ((1.0 - alpha) * CC + 2.0 * alpha", "return (CC + 2.0 * alpha", "dropped (1 - alpha)"),
    ("gw.py", "fgw_grad_prescribed", "- 4.0 * alpha * triple_product_dense(x, y, T, k))", "- 4.0 * triple_product_dense(x, y, T, k))", "dropped alpha on the product"),
    ("gw.py", "fgw_grad_prescribed", "CC = (fx[:, None] - fy[None, :]) ** 2\n    c, c2", "CC = np.abs(fx[:, None] - fy[None, :])\n    c, c2", "feature cost not squared"),
    ("gw.py", "fgw_objective", "return float((1.0 - alpha) * np.sum(CC * T) + alpha * objective", "return float(np.sum(CC * T) + alpha * objective", "dropped (1 - alpha)"),
    ("gw.py", "fgw_objective", "+ alpha * objective(x, y, T, k))", "+ objective(x, y, T, k))", "dropped alpha"),
    ("solver.py", "logsumexp", "s = np.sum(np.exp(a - m), axis=axis, keepdims=True)", "s = np.sum(np.exp(a), axis=axis, keepdims=True)", "shift not applied inside"),
    ("solver.py", "plan_from_duals", "np.exp((f[:, None] + g[None, :] - np.asarray(G, np.float64)) / eps)", "np.exp((f[:, None] - g[None, :] - np.asarray(G, np.float64)) / eps)", "sign of g"),
    ("solver.py", "sinkhorn", "f = eps * lp - eps * logsumexp((g[None, :] - G) / eps, axis=1)", "f = eps * lp - eps * logsumexp((g[None, :] + G) / eps, axis=1)", "sign of the cost"),
    ("solver.py", "sinkhorn", "g = eps * lq - eps * logsumexp((f[:, None] - G) / eps, axis=0)", "g = eps * lp - eps * logsumexp((f[:, None] - G) / eps, axis=0)", "ln p in the g-update"),
    ("solver.py", "sinkhorn", "g = eps * lq - eps * logsumexp((f[:, None] - G) / eps, axis=0)", "g = lq - eps * logsumexp((f[:, None] - G) / eps, axis=0)", "eps missing on ln q"),
    ("solver.py", "sinkhorn", "if tol is not None and used % check_every == 0:", "if tol is not None and it % check_every == 0:", "check schedule off by one"),
    ("solver.py", "entropic_gw", "f, g, used = sinkhorn(G, p, q, tau, counts[l], f, g, tol=tol, check_every=check_every)\n        T = plan_from_duals(G, f, g, tau)\n        if tau != eps:\n            lnT = (f[:, None] + g[None, :] - G) / tau\n        out[\"E\"].append(objective(", "f, g, used = sinkhorn(G, p, q, tau, counts[l], None, None, tol=tol, check_every=check_every)\n        T = plan_from_duals(G, f, g, tau)\n        if tau != eps:\n            lnT = (f[:, None] + g[None, :] - G) / tau\n        out[\"E\"].append(objective(", "cold-started duals (reading R7)"),
    ("solver.py", "entropic_gw", "G = G + (eps - tau) * lnT  # the cost Pi", "G = G + (tau - eps) * lnT  # the cost Pi", "sign of the tau term"),
    ("solver.py", "entropic_gw", 'out["entropic_objective"] = out["gw_objective"] + eps * entropy(T)\n    return out\n\n\ndef entropic_fgw', 'out["entropic_objective"] = out["gw_objective"] - eps * entropy(T)\n    return out\n\n\ndef entropic_fgw', "sign of the entropy term"),
    ("solver.py", "entropic_gw", "T = np.outer(p, q) if T0 is None else np.array(T0, dtype=np.float64)\n    f = np.zeros(x.size)\n    g = np.zeros(y.size)\n    counts = [int(inner)] * outer if np.isscalar(inner) else [int(c) for c in inner]\n    out = {\"E\": [], \"viol\": [], \"inner_used\": [], \"G\": []}", "T = np.outer(p, q)\n    f = np.zeros(x.size)\n    g = np.zeros(y.size)\n    counts = [int(inner)] * outer if np.isscalar(inner) else [int(c) for c in inner]\n    out = {\"E\": [], \"viol\": [], \"inner_used\": [], \"G\": []}", "T0 ignored"),
    ("solver.py", "entropic_gw", "T = plan_from_duals(G, f, g, tau)\n        if tau != eps:\n            lnT = (f[:, None] + g[None, :] - G) / tau\n        out[\"E\"].append(objective(x, y, T, k))", "T = plan_from_duals(G, f, g, eps)\n        if tau != eps:\n            lnT = (f[:, None] + g[None, :] - G) / tau\n        out[\"E\"].append(objective(x, y, T, k))", "plan at eps instead of tau"),
    ("solver.py", "entropic_fgw", 'out["E"].append(fgw_objective(x, y, fx, fy, alpha, T, k))', 'out["E"].append(objective(x, y, T, k))', "FGW trace reports the GW part only"),
    ("solver.py", "entropic_fgw", "G = fgw_grad_prescribed(x, y, p, q, fx, fy, alpha, T, k)", "G = fgw_grad_prescribed(x, y, p, q, fx[::-1], fy, alpha, T, k)", "feature vector reversed"),
    ("grid2d.py", "grid_points", 'A, B = np.meshgrid(s, s, indexing="ij")', 'A, B = np.meshgrid(s, s, indexing="xy")', "flattening order"),
    ("grid2d.py", "dist2d", "+ np.abs(P[:, None, 1] - P[None, :, 1])\n    return man ** k", "+ np.abs(P[:, None, 1] - P[None, :, 1]) ** 2\n    return man ** k", "second axis squared"),
    ("grid2d.py", "apply_distance_2d", "out += math.comb(k, r) * (D1 ** r) @ V @ (D1 ** (k - r)).T", "out += (D1 ** r) @ V @ (D1 ** (k - r)).T", "dropped binomial"),
    ("grid2d.py", "grad_prescribed_2d", "return 2.0 * (c[:, None] + c2[None, :]) - 4.0 * (DX @ T @ DY)", "return 2.0 * (c[:, None] + c2[None, :]) - 4.0 * (DX @ T @ DX[:T.shape[1], :T.shape[1]])" , "D_X on the right"),
    ("grid2d.py", "objective_2d", "- 2.0 * np.sum((DX @ T @ DY) * T))", "- 4.0 * np.sum((DX @ T @ DY) * T))", "cross term factor"),
    ("grid2d.py", "fgw_grad_prescribed_2d", "return (1.0 - alpha) * CC + alpha * grad_prescribed_2d", "return CC + alpha * grad_prescribed_2d", "dropped (1 - alpha)"),
    ("grid2d.py", "fgw_objective_2d", "return float((1.0 - alpha) * np.sum(CC * T) + alpha * objective_2d", "return float(np.sum(CC * T) + alpha * objective_2d", "dropped (1 - alpha)"),
    ("grid2d.py", "entropic_gw_2d", "f, g, _used = sinkhorn(G, p, q, eps, inner, f, g)\n        T = plan_from_duals(G, f, g, eps)\n        out[\"E\"].append(objective_2d(", "f, g, _used = sinkhorn(G, q, p, eps, inner, f, g)\n        T = plan_from_duals(G, f, g, eps)\n        out[\"E\"].append(objective_2d(", "marginals swapped"),
    ("ugw.py", "kl", "return float(np.sum(_xlogy(x, y)) - x.sum() + y.sum())", "return float(np.sum(_xlogy(x, y)) - x.sum())", "dropped m(y)"),
    ("ugw.py", "kl_tensor_sq", "2.0 * x.sum() * np.sum(_xlogy(x, y)) - x.sum() ** 2 + y.sum() ** 2", "x.sum() * np.sum(_xlogy(x, y)) - x.sum() ** 2 + y.sum() ** 2", "dropped factor 2"),
    ("ugw.py", "ugw_functional", "+ rho * kl_tensor_sq(b, v)", "+ rho * kl_tensor_sq(a, v[:a.size] if v.size >= a.size else u)", "second marginal term wrong"),
    ("ugw.py", "ugw_cost", "half = 0.5 * grad_prescribed(x, y, a, b, Gh, k)", "half = grad_prescribed(x, y, a, b, Gh, k)", "dropped the 1/2"),
    ("ugw.py", "ugw_cost", "gsc = (rho * np.sum(_xlogy(a, u)) + rho * np.sum(_xlogy(b, v))", "gsc = (rho * np.sum(_xlogy(a, u)) + eps * np.sum(_xlogy(b, v))", "eps for rho"),
    ("ugw.py", "unbalanced_plan", "* np.outer(_f64(u), _f64(v))", "", "dropped the reference measure"),
    ("ugw.py", "unbalanced_sinkhorn", "kap = rho_t / (rho_t + eps_t)", "kap = eps_t / (rho_t + eps_t)", "wrong damping factor"),
    ("ugw.py", "unbalanced_sinkhorn", "g = -kap * eps_t * logsumexp((f[:, None] - C) / eps_t + lu[:, None], axis=0)", "g = -kap * eps_t * logsumexp((f[:, None] - C) / eps_t, axis=0)", "dropped ln u"),
    ("ugw.py", "entropic_ugw", "G = math.sqrt(mh / Gn.sum()) * Gn", "G = (mh / Gn.sum()) * Gn", "mass rescaling without the root"),
    ("ugw.py", "entropic_ugw", "f, g = unbalanced_sinkhorn(C, u, v, mh * rho, mh * eps, inner, f, g)", "f, g = unbalanced_sinkhorn(C, u, v, rho, mh * eps, inner, f, g)", "rho not scaled by the mass"),
    ("streamed.py", "const_term_blocked", "** (2 * k)) @ w", "** k) @ w", "c at power k"),
    ("streamed.py", "grad_rows_cols", "V[j0:j1] = Tb @ DYJ", "V[j0:j1] = Tb @ DYJ[::-1]", "reversed D_Y block"),
    ("streamed.py", "grad_rows_cols", "GI = 2.0 * (c[I, None] + c2[None, :]) - 4.0 * R", "GI = 2.0 * (c[I, None] + c2[None, :]) - 2.0 * R", "rows: factor on the product"),
    ("streamed.py", "grad_rows_cols", "GJ = 2.0 * (c[:, None] + c2[None, J]) - 4.0 * Cc", "GJ = 2.0 * (c[:, None] + c2[None, :][:, :J.size]) - 4.0 * Cc", "columns: c' not indexed by J"),
    ("streamed.py", "marginals_streamed", "b += Tb.sum(axis=0)", "b = Tb.sum(axis=0)", "column sums not accumulated"),
    ("streamed.py", "violation_streamed", "return float(max(np.max(np.abs(a - p)), np.max(np.abs(b - q))))", "return float(np.max(np.abs(a - p)))", "rows only"),
    ("streamed.py", "dist_apply_prefix", "out = s * (2.0 * P - Pt) - (2.0 * Q - Qt)", "out = s * (2.0 * P - Pt) - (2.0 * Q + Qt)", "sign of the total"),
    ("streamed.py", "objective_k1", "carry.append((b.copy(), bx.copy()))", "carry.append((b, bx))", "carry aliases the running total"),
    ("streamed.py", "objective_k1", "return 2.0 * (m0 * m2 - m1 * m1)", "return 2.0 * (m0 * m2 + m1 * m1)", "sign in the moment expansion"),
    ("streamed.py", "objective_k1", "return float(quad(x, a) + quad(y, b) - 2.0 * total)", "return float(quad(x, a) + quad(y, b) - total)", "cross term factor"),
]


def run_one(idx, mut):
    fname, fn, old, new, what = mut
    tmp = tempfile.mkdtemp(prefix="mut%02d_" % idx)
    try:
        for d in ("oracle", "tests", "workloads"):
            shutil.copytree(os.path.join(ROOT, d), os.path.join(tmp, d))
        path = os.path.join(tmp, "oracle", fname)
        src = open(path).read()
        if src.count(old) < 1:
            return idx, mut, "NOT APPLIED (text not found)"
        open(path, "w").write(src.replace(old, new, 1))
        r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                            "tests/test_oracle_pins.py", "tests/test_oracle_ugw.py"],
                           cwd=tmp, capture_output=True, text=True, timeout=1800)
        tail = [l for l in r.stdout.strip().splitlines() if l.strip()]
        first_fail = next((l for l in tail if l.startswith("FAILED") or l.startswith("ERROR")), "")
        return idx, mut, ("killed: " + first_fail[:110]) if r.returncode != 0 else "SURVIVED"
    finally:
        shutil.rmtree(tmp, ignore_errors=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--jobs", type=int, default=8)
    ap.add_argument("--only", default=None, help="comma-separated substrings of 'function: mistake' to select mutations")
    a = ap.parse_args()
    muts = list(MUTATIONS)
    if a.only:
        keys = [k.strip() for k in a.only.split(",")]
        muts = [m for m in muts if any(k in "%s: %s" % (m[1], m[4]) for k in keys)]
        if not muts:
            print("no mutation selected")
            return 2
    res = []
    with cf.ThreadPoolExecutor(a.jobs) as ex:
        for r in ex.map(lambda im: run_one(*im), enumerate(muts)):
            res.append(r)
            idx, (fname, fn, old, new, what), verdict = r
            print("%2d  oracle/%-11s %-24s %-40s %s" % (idx, fname, fn, what[:40], verdict), flush=True)
    surv = [r for r in res if r[2] == "SURVIVED"]
    na = [r for r in res if r[2].startswith("NOT")]
    print("mutations %d, killed %d, survived %d, not applied %d" %
          (len(res), len(res) - len(surv) - len(na), len(surv), len(na)))
    return 1 if surv or na else 0


if __name__ == "__main__":
    sys.exit(main())
