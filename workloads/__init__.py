"""Seeded synthetic input generators (shared by tests, bench.py and smoke()).

This module holds NONE of the method's arithmetic: it only draws supports,
marginals and plans with NumPy's PCG64 (``default_rng(seed)``, reading R20) in
the order SURVEY.md §8(d) lists, so that the CUDA path and the oracle receive
identical float64 arrays.  BASELINE.json names no public dataset; every config
is synthetic (the paper's own hot-path workload, is too).

Configs (BASELINE.json ``configs``):
  C1  1-D entropic GW, N=M=256, Uniform[0,1) sorted, uniform p,q, eps=1e-2, 20x100
  C2  N=M=4096, 3-component Gaussian mixture x, y = 1 - x + N(0, 1e-3^2), Dirichlet(1) p,q, eps=5e-3
  C3  gradient only, N=M=16384, T = Exp(1) entries rescaled to uniform marginals
  C4  N=M=65536, Uniform[0,1) sorted, uniform p,q, eps=1e-3, 10 outer x 100 inner
  C5  FGW N=32768, M=24576, Beta(2,5)/Beta(5,2) supports, N(0,1) features, Dirichlet(0.5), alpha=0.5
  T2  the paper's Table 2 GW workload: uniform grid x_i=(i-1)/(N-1), U[0,1] weights normalised
"""

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

__all__ = ["Problem", "config1", "config2", "config3", "config4", "config5",
           "table2", "uniform_problem", "random_plan", "CONFIGS"]


@dataclass
class Problem:
    name: str
    x: np.ndarray          # (N,) float64, non-decreasing
    y: np.ndarray          # (M,) float64, non-decreasing
    p: np.ndarray          # (N,) float64, >= 0, sums to 1
    q: np.ndarray          # (M,) float64
    eps: float = 1e-2
    outer: int = 10
    inner: int = 100
    fx: Optional[np.ndarray] = None   # FGW features (C5)
    fy: Optional[np.ndarray] = None
    alpha: float = 1.0
    rho: Optional[float] = None
    extra: dict = field(default_factory=dict)

    @property
    def n(self):
        return self.x.size

    @property
    def m(self):
        return self.y.size


def _normalise(w):
    w = np.asarray(w, dtype=np.float64)
    return w / w.sum()


def uniform_problem(n, m=None, seed=0, eps=1e-2, outer=10, inner=100, name="uniform"):
    """x, y ~ sort(Uniform[0,1)), uniform marginals (the C1/C4 recipe at any size)."""
    m = n if m is None else m
    rng = np.random.default_rng(seed)
    x = np.sort(rng.random(n))
    y = np.sort(rng.random(m))
    return Problem(name, x, y, np.full(n, 1.0 / n), np.full(m, 1.0 / m), eps, outer, inner)


def config1(seed=0):
    """C1: N=M=256, eps=1e-2, T0 = p (x) q, 20 outer x 100 Sinkhorn, seed 0."""
    return uniform_problem(256, 256, seed, eps=1e-2, outer=20, inner=100, name="C1")


def config2(n=4096, seed=0):
    """C2 (reading R21): means (0.2, 0.5, 0.8), sigma 0.05;
    y = sort(1 - x + 1e-3 N(0,1)); p, q ~ Dirichlet(1); eps = 5e-3; 20 outer (R9)."""
    rng = np.random.default_rng(seed)
    comp = rng.choice(3, n)
    x = np.sort(np.array([0.2, 0.5, 0.8])[comp] + 0.05 * rng.standard_normal(n))
    y = np.sort(1.0 - x + 1e-3 * rng.standard_normal(n))
    p = rng.dirichlet(np.ones(n))
    q = rng.dirichlet(np.ones(n))
    return Problem("C2", x, y, p, q, eps=5e-3, outer=20, inner=100)


def random_plan(n, m, p, q, rng, rescalings=50, dtype=np.float32):
    """Exp(1) entries, then `rescalings` alternating row -> column rescalings in
    float64 towards (p, q), cast to `dtype` (reading R22).  The cast
    array is the shared input: both sides read the same values."""
    Z = rng.exponential(size=(n, m))
    for _ in range(rescalings):
        Z *= (p / Z.sum(axis=1))[:, None]
        Z *= (q / Z.sum(axis=0))[None, :]
    return Z.astype(dtype)


def config3(n=16384, seed=0, rescalings=50):
    """C3: gradient only; x, y sorted uniform; p = q uniform; T from `random_plan`."""
    rng = np.random.default_rng(seed)
    x = np.sort(rng.random(n))
    y = np.sort(rng.random(n))
    p = np.full(n, 1.0 / n)
    q = np.full(n, 1.0 / n)
    prob = Problem("C3", x, y, p, q)
    prob.extra["T"] = random_plan(n, n, p, q, rng, rescalings)
    return prob


def config4(n=65536, seed=0):
    """C4: N=M=65536 (or a smaller n with the same recipe), eps=1e-3, 10 outer x 100 inner."""
    return uniform_problem(n, n, seed, eps=1e-3, outer=10, inner=100, name="C4")


def config5(n=32768, m=24576, seed=0):
    """C5: x ~ sort Beta(2,5), y ~ sort Beta(5,2); fx, fy ~ N(0,1);
    p ~ Dirichlet(0.5), q ~ Dirichlet(0.5); alpha = 0.5; rho = 1.0; eps = 1e-2 (R12)."""
    rng = np.random.default_rng(seed)
    x = np.sort(rng.beta(2.0, 5.0, n))
    y = np.sort(rng.beta(5.0, 2.0, m))
    fx = rng.standard_normal(n)
    fy = rng.standard_normal(m)
    p = rng.dirichlet(0.5 * np.ones(n))
    q = rng.dirichlet(0.5 * np.ones(m))
    return Problem("C5", x, y, p, q, eps=1e-2, outer=20, inner=100, fx=fx, fy=fy,
                   alpha=0.5, rho=1.0)


def table2(n, seed=0, eps=0.002, outer=10, inner=100):
    """The paper's Table 2 GW workload: uniform grid
    x_i = y_i = (i-1)/(N-1), weights U[0,1] normalised, k = 1, eps = 0.002, 10 outer."""
    rng = np.random.default_rng(seed)
    grid = np.arange(n, dtype=np.float64) / max(n - 1, 1)
    p = _normalise(rng.random(n))
    q = _normalise(rng.random(n))
    return Problem("T2", grid.copy(), grid.copy(), p, q, eps=eps, outer=outer, inner=inner)


CONFIGS = {"C1": config1, "C2": config2, "C3": config3, "C4": config4, "C5": config5}
