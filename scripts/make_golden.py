#!/usr/bin/env python
"""Write oracle-only golden trajectories used by the GPU parity tests (tier rules ③: a stored
expected value is written by a committed script that calls only oracle/).

    python scripts/make_golden.py c2        # C2 at its full size N = M = 4096 (~10 min on 8+ cores)
    python scripts/make_golden.py c4_16384  # C4's recipe at N = M = 16384 (~1.5 h on 8 cores)

Output: tests/golden/<name>.json with the oracle's objective E(T^l) for every outer iteration,
the final entropic objective and the final marginal violation, plus the recipe it ran.
"""

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
import workloads as W  # noqa: E402


def c2():
    P = W.config2(4096)
    t0 = time.time()
    ro = O.entropic_gw(P.x, P.y, P.p, P.q, P.eps, 20, 100)
    return {"name": "c2_n4096_trajectory", "recipe": "workloads.config2(4096): BASELINE configs[1] at full size, "
            "eps=5e-3, T0=p(x)q, 20 outer x 100 inner (readings R7, R9), seed 0",
            "E": [float(e) for e in ro["E"]], "viol": [float(v) for v in ro["viol"]],
            "gw_objective": float(ro["gw_objective"]), "entropic_objective": float(ro["entropic_objective"]),
            "oracle_seconds": time.time() - t0}


def c4_16384():
    """SURVEY §8(c) C4 parity (i): the C4 recipe (eps = 1e-3, fixed K = 100, 10 outer) at N = M = 16384."""
    P = W.config4(16384)
    t0 = time.time()
    ro = O.entropic_gw(P.x, P.y, P.p, P.q, P.eps, 10, 100)
    return {"name": "c4_n16384_trajectory", "recipe": "workloads.config4(16384): BASELINE configs[3]'s recipe "
            "at N = M = 16384, eps=1e-3, T0=p(x)q, 10 outer x 100 inner (readings R7, R8, R9), seed 0",
            "E": [float(e) for e in ro["E"]], "viol": [float(v) for v in ro["viol"]],
            "gw_objective": float(ro["gw_objective"]), "entropic_objective": float(ro["entropic_objective"]),
            "oracle_seconds": time.time() - t0}


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "c2"
    out = {"c2": c2, "c4_16384": c4_16384}[which]()
    path = os.path.join(ROOT, "tests", "golden", out["name"] + ".json")
    json.dump(out, open(path, "w"), indent=1)
    print("wrote", path, "in %.0f s" % out["oracle_seconds"])
