"""Plain, slow, float64 CPU oracle for the FGC entropic Gromov-Wasserstein hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import anything
from this package.  The product path (``paper_2404_08970_b200``) never imports it,
and this package never imports the product path, torch, or any shared helper:
it is NumPy float64 written from the paper (arXiv 2404.08970, ``PAPER.md``).

Every function cites the passage it follows.  "PAPER.md:N" is a line of the
paper's LaTeX source; "SPEC.md:N" a line of the CPU-program spec written from it.

Pins (tests/test_oracle_*.py, ``-m "not gpu"``) tie each function to something
other than itself: worked examples (tests/golden/), closed forms, brute force,
invariants and finite differences.  Functions without such a pin would say
"parity unpinned".  ``ugw`` (Remark 3) follows readings R32-R35 (the paper leaves g(G^)
undefined): its pieces are pinned (finite differences of the functional,
direct minimisation of the subproblem, the balanced rho -> infinity limit) and so is the loop's
fixed point (a critical point of the functional Remark 3 minimises); the per-iteration trajectory
of the reading has no worked example in the paper and is parity unpinned.
"""

from .gw import (  # noqa: F401
    dist,
    const_term,
    grad_entrywise,
    grad_prescribed,
    grad_prescribed_dp,
    grad_realized,
    ref_dp_lower,
    ref_dp_upper,
    ref_dp_distance,
    triple_product_dp,
    triple_product_dense,
    objective,
    objective_bruteforce,
    entropy,
    violation,
    fgw_grad_prescribed,
    fgw_objective,
)
from .solver import (  # noqa: F401
    logsumexp,
    sinkhorn,
    entropic_gw,
    entropic_fgw,
    plan_from_duals,
)
from .grid2d import (  # noqa: F401
    grid_points,
    dist2d,
    apply_distance_2d,
    grad_prescribed_2d,
    fgw_grad_prescribed_2d,
    fgw_objective_2d,
    entropic_fgw_2d,
    objective_2d,
    entropic_gw_2d,
)
from .ugw import (  # noqa: F401
    kl,
    kl_tensor_sq,
    ugw_functional,
    ugw_functional_bruteforce,
    ugw_cost,
    unbalanced_sinkhorn,
    unbalanced_plan,
    entropic_ugw,
)
from .streamed import (  # noqa: F401
    const_term_blocked,
    grad_rows_cols,
    marginals_streamed,
    violation_streamed,
    objective_k1,
    dist_apply_prefix,
    fgw_rows_cols,
    fgw_objective_k1,
    ugw_functional_k1,
)
