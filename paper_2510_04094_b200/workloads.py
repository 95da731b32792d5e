"""Seeded synthetic ODE instances for the five BASELINE.json configurations.

The reference ships no generator for these configs ("no reference
test pins them"), so this module is the single source of inputs for the oracle,
the CUDA path, the tests and ``bench.py``.  It follows SURVEY.md §8(d):

* ``rng = np.random.default_rng([config_id, seed, instance])``, draws in the
  fixed order documented in :func:`_draw_linear` / :func:`_draw_nonlinear`.
* manufactured solution ``y*(t) = sum_k A_k sin(w_k t + phi_k)`` with
  ``A ~ U[0.5, 1.5]``, ``w ~ U[1, 10]``, ``phi ~ U[0, 2 pi]``; K = 3 (c0, c3),
  5 (c1, c2), 7 (c4).
* ``a(t) = a0 + a1 sin(2 pi t)``, ``a0 ~ U[0.5, 2]``, ``a1 ~ U[-0.5, 0.5]``;
  ``b(t) = b0 + b1 sin(2 pi t)``, ``b0 ~ U[0.6, 2]``, ``b1 ~ U[-0.5, 0.5]``
  (so ``b >= 0.1`` as BASELINE.json asks — builder decision, recorded in DESIGN.md).
* canonical form of the reference (``pkg/src/nysode/problems.py:3-6``):
  ``y^(p) = sum_k f_k y^(p-k) + r`` so ``f_1 = -a``, ``f_2 = -b``, ``r = f``.
* IVP conditions ``y(0) = y*(0)`` (and ``y'(0) = y*'(0)`` for p = 2).
* "RBF sigma" is mapped to the reference's ``sigma2 = sigma**2``
  (``pkg/src/nysode/kernel.py:69-72``; SURVEY.md §8d ambiguity 1).

Nothing here touches the GPU; the arrays it emits are what crosses the C-ABI.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

TWO_PI = 2.0 * math.pi


@dataclass(frozen=True)
class ConfigSpec:
    """One BASELINE.json configuration (index = position in ``configs``)."""

    cid: int
    n: int
    m: int
    domain: tuple[float, float]
    order: int
    terms: int
    gamma: float
    sigma: float            # RBF sigma; sigma2 = sigma**2
    batch: int = 1
    nonlinear: bool = False
    newton_max_iters: int = 20
    note: str = ""

    @property
    def sigma2(self) -> float:
        return self.sigma * self.sigma

    @property
    def n_c(self) -> int:   # IVP constraint rows t_2..t_n (pkg/src/nysode/linear.py:66-68)
        return self.n - 1


# sigma choices: c0 and c3 are fixed by BASELINE.json (sigma = 0.1).  c1 and c4
# are "tuned per seed from [0.05, 0.5]"; c2 needs one shared sigma because the
# landmarks are shared.  The tuning rule (oracle/tune_sigma.py) is an
# oracle-side grid search over SIGMA_CANDIDATES minimising the relative L2
# error vs y*, restricted to sigmas whose oracle error is reproducible: swapping
# LAPACK's eigensolver driver (dsyevd -> dsyev) must move the error vs y* by
# < 1e-3 of itself, i.e. 10x inside the north star's 1 % error gate.  Without
# that guard the 1 % gate is unattainable even for the reference against
# itself (c2 sigma=0.3: 300 % swing).  Outcome (frozen here):
# c1 -> 0.4 (m_eff 50), c2 -> 0.1 (m_eff 64 = m), c4 -> 0.5 (m_eff 256).
SIGMA_CANDIDATES = (0.05, 0.1, 0.15, 0.2, 0.3, 0.4, 0.5)

CONFIGS: dict[int, ConfigSpec] = {
    0: ConfigSpec(0, n=1000, m=20, domain=(0.0, 1.0), order=1, terms=3,
                  gamma=1e8, sigma=0.1),
    1: ConfigSpec(1, n=10_000, m=50, domain=(0.0, 5.0), order=2, terms=5,
                  gamma=1e9, sigma=0.4),
    2: ConfigSpec(2, n=4096, m=64, domain=(0.0, 2.0), order=2, terms=5,
                  gamma=1e9, sigma=0.1, batch=4096),
    3: ConfigSpec(3, n=2000, m=40, domain=(0.0, 1.0), order=1, terms=3,
                  gamma=1e8, sigma=0.1, batch=256, nonlinear=True),
    4: ConfigSpec(4, n=1 << 22, m=256, domain=(0.0, 100.0), order=2, terms=7,
                  gamma=1e9, sigma=0.5),
}


# ---------------------------------------------------------------------------
# manufactured solutions


@dataclass(frozen=True)
class SinusoidSum:
    """y*(t) = sum_k A_k sin(w_k t + phi_k) and its analytic derivatives."""

    amp: np.ndarray
    freq: np.ndarray
    phase: np.ndarray

    def deriv(self, t, order: int = 0) -> np.ndarray:
        t = np.asarray(t, dtype=float)
        out = np.zeros_like(t)
        # d^q/dt^q sin(x) = sin(x + q pi/2)
        for a, w, ph in zip(self.amp, self.freq, self.phase):
            out = out + a * w ** order * np.sin(w * t + ph + order * (math.pi / 2))
        return out

    def __call__(self, t) -> np.ndarray:
        return self.deriv(t, 0)


@dataclass(frozen=True)
class LinearInstance:
    """One linear IVP in canonical form y^(p) = sum_k f_k y^(p-k) + r."""

    cid: int
    seed: int
    index: int
    order: int
    domain: tuple[float, float]
    sol: SinusoidSum
    a: tuple[float, float]                    # a0, a1
    b: Optional[tuple[float, float]] = None   # b0, b1 (order 2 only)

    def a_fn(self, t):
        t = np.asarray(t, dtype=float)
        return self.a[0] + self.a[1] * np.sin(TWO_PI * t)

    def b_fn(self, t):
        t = np.asarray(t, dtype=float)
        return self.b[0] + self.b[1] * np.sin(TWO_PI * t)

    def coeff_fns(self) -> tuple[Callable, ...]:
        """(f_1, ..., f_p) of the canonical form (problems.py:3-6)."""
        if self.order == 1:
            return (lambda t: -self.a_fn(t),)
        return (lambda t: -self.a_fn(t), lambda t: -self.b_fn(t))

    def forcing_fn(self, t):
        t = np.asarray(t, dtype=float)
        if self.order == 1:
            return self.sol.deriv(t, 1) + self.a_fn(t) * self.sol(t)
        return (self.sol.deriv(t, 2) + self.a_fn(t) * self.sol.deriv(t, 1)
                + self.b_fn(t) * self.sol(t))

    def conditions(self) -> list[tuple[float, int, float]]:
        """IVP entries (point, derivative order, value) at t_1."""
        t0 = float(self.domain[0])
        out = [(t0, 0, float(self.sol(np.array([t0]))[0]))]
        if self.order == 2:
            out.append((t0, 1, float(self.sol.deriv(np.array([t0]), 1)[0])))
        return out

    def sample(self, pts: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
        """Coefficient rows f_k(pts) (p x n_c) and forcing r(pts) (n_c,)."""
        coef = np.stack([np.asarray(f(pts), dtype=float) for f in self.coeff_fns()])
        return coef, np.asarray(self.forcing_fn(pts), dtype=float)


@dataclass(frozen=True)
class NonlinearInstance:
    """First-order IVP y' = f(t, y) for config 3.

    kind "quad": f = -k y^2 + g(t), g = y*' + k y*^2, f_y = -2 k y, f_yy = -2 k
    kind "sin" : f = sin(y) + g(t), g = y*' - sin(y*), f_y = cos y, f_yy = -sin y
    (SURVEY.md §8d).  Even instances are "quad", odd instances are "sin".
    """

    cid: int
    seed: int
    index: int
    kind: str
    k: float
    domain: tuple[float, float]
    sol: SinusoidSum

    def g_fn(self, t):
        t = np.asarray(t, dtype=float)
        ys, dys = self.sol(t), self.sol.deriv(t, 1)
        if self.kind == "quad":
            return dys + self.k * ys * ys
        return dys - np.sin(ys)

    def rhs(self, t, y):
        y = np.asarray(y, dtype=float)
        if self.kind == "quad":
            return -self.k * y * y + self.g_fn(t)
        return np.sin(y) + self.g_fn(t)

    def rhs_y(self, t, y):
        y = np.asarray(y, dtype=float)
        if self.kind == "quad":
            return -2.0 * self.k * y
        return np.cos(y)

    def rhs_yy(self, t, y):
        y = np.asarray(y, dtype=float)
        if self.kind == "quad":
            return np.full_like(y, -2.0 * self.k)
        return -np.sin(y)

    def conditions(self) -> list[tuple[float, int, float]]:
        t0 = float(self.domain[0])
        return [(t0, 0, float(self.sol(np.array([t0]))[0]))]

    # device-side description of f: f(t, y) = g(t) + quad * y^2 + sin_c * sin(y)
    @property
    def quad_coeff(self) -> float:
        return -self.k if self.kind == "quad" else 0.0

    @property
    def sin_coeff(self) -> float:
        return 1.0 if self.kind == "sin" else 0.0


@dataclass(frozen=True)
class NonlinearInstance2:
    """Second-order IVP y'' = f(t, y, y') -- the SURVEY.md §8f next-row-2 shape
    (the catalog's P14/P15 are second-order nonlinear BVPs), manufactured like
    config 3:

    kind "drag": f = -k (y')^2 + g(t),      g = y*'' + k (y*')^2
    kind "pend": f = -sin(y) - k y' + g(t), g = y*'' + sin(y*) + k y*'
    Even instances are "drag", odd ones "pend"; conditions y(t0), y'(t0).
    """

    seed: int
    index: int
    kind: str
    k: float
    domain: tuple[float, float]
    sol: SinusoidSum

    def g_fn(self, t):
        t = np.asarray(t, dtype=float)
        ys, d1, d2 = self.sol(t), self.sol.deriv(t, 1), self.sol.deriv(t, 2)
        if self.kind == "drag":
            return d2 + self.k * d1 * d1
        return d2 + np.sin(ys) + self.k * d1

    def rhs(self, t, y, yp):
        y, yp = np.asarray(y, dtype=float), np.asarray(yp, dtype=float)
        if self.kind == "drag":
            return -self.k * yp * yp + self.g_fn(t)
        return -np.sin(y) - self.k * yp + self.g_fn(t)

    def rhs_y(self, t, y, yp):
        y = np.asarray(y, dtype=float)
        return np.zeros_like(y) if self.kind == "drag" else -np.cos(y)

    def rhs_yp(self, t, y, yp):
        yp = np.asarray(yp, dtype=float)
        return -2.0 * self.k * yp if self.kind == "drag" else np.full_like(yp, -self.k)

    def rhs_yy(self, t, y, yp):
        y = np.asarray(y, dtype=float)
        return np.zeros_like(y) if self.kind == "drag" else np.sin(y)

    def rhs_yyp(self, t, y, yp):
        return np.zeros_like(np.asarray(y, dtype=float))

    def rhs_ypyp(self, t, y, yp):
        y = np.asarray(y, dtype=float)
        return np.full_like(y, -2.0 * self.k) if self.kind == "drag" else np.zeros_like(y)

    def second_partials(self) -> dict:
        return {(0, 0): self.rhs_yy, (0, 1): self.rhs_yyp, (1, 1): self.rhs_ypyp}

    def conditions(self) -> list[tuple[float, int, float]]:
        t0 = np.array([float(self.domain[0])])
        return [(float(t0[0]), 0, float(self.sol(t0)[0])),
                (float(t0[0]), 1, float(self.sol.deriv(t0, 1)[0]))]


# second-order nonlinear workload (tests): n, m, sigma, gamma of the c3 scale
NONLINEAR2 = dict(n=400, m=40, domain=(0.0, 1.0), terms=3, gamma=1e8, sigma=0.2,
                  newton_max_iters=30)


def nonlinear2_instance(seed: int = 0, index: int = 0) -> NonlinearInstance2:
    # draw order: A[K], w[K], phi[K], k  (rng seeded by [5, seed, index])
    rng = np.random.default_rng([5, seed, index])
    sol = _draw_solution(rng, NONLINEAR2["terms"])
    k = float(rng.uniform(0.2, 1.0))
    kind = "drag" if index % 2 == 0 else "pend"
    return NonlinearInstance2(seed, index, kind, k, NONLINEAR2["domain"], sol)


def _draw_solution(rng: np.random.Generator, terms: int) -> SinusoidSum:
    amp = rng.uniform(0.5, 1.5, size=terms)
    freq = rng.uniform(1.0, 10.0, size=terms)
    phase = rng.uniform(0.0, TWO_PI, size=terms)
    return SinusoidSum(amp, freq, phase)


def _draw_linear(cfg: ConfigSpec, seed: int, index: int) -> LinearInstance:
    # draw order: A[K], w[K], phi[K], a0, a1, (b0, b1)
    rng = np.random.default_rng([cfg.cid, seed, index])
    sol = _draw_solution(rng, cfg.terms)
    a = (float(rng.uniform(0.5, 2.0)), float(rng.uniform(-0.5, 0.5)))
    b = None
    if cfg.order == 2:
        b = (float(rng.uniform(0.6, 2.0)), float(rng.uniform(-0.5, 0.5)))
    return LinearInstance(cfg.cid, seed, index, cfg.order, cfg.domain, sol, a, b)


def _draw_nonlinear(cfg: ConfigSpec, seed: int, index: int) -> NonlinearInstance:
    # draw order: A[K], w[K], phi[K], k
    rng = np.random.default_rng([cfg.cid, seed, index])
    sol = _draw_solution(rng, cfg.terms)
    k = float(rng.uniform(0.5, 2.0))
    kind = "quad" if index % 2 == 0 else "sin"
    return NonlinearInstance(cfg.cid, seed, index, kind, k, cfg.domain, sol)


def instance(cid: int, seed: int = 0, index: int = 0, cfg: Optional[ConfigSpec] = None):
    cfg = cfg or CONFIGS[cid]
    if cfg.nonlinear:
        return _draw_nonlinear(cfg, seed, index)
    return _draw_linear(cfg, seed, index)


def grid(cfg: ConfigSpec) -> np.ndarray:
    """Uniform collocation grid, built on host (never on device)."""
    return np.linspace(cfg.domain[0], cfg.domain[1], cfg.n)


def equidistant_landmarks(grid_pts: np.ndarray, m: int) -> np.ndarray:
    """Equidistant subsample idx = round(i (n-1)/(m-1)) (nystrom.py:90-91)."""
    n = grid_pts.size
    idx = np.round(np.arange(m) * (n - 1) / (m - 1)).astype(int)
    return grid_pts[idx]


@dataclass
class LinearBatch:
    """Sampled arrays for B linear instances sharing grid and landmarks.

    coef    (B, p, n_c)   f_k at the constraint points, k = 1..p
    forcing (B, n_c)      r at the constraint points
    cond_values (B, p)    IVP values; condition points/orders are shared
    """

    cfg: ConfigSpec
    grid: np.ndarray
    landmarks: np.ndarray
    pts: np.ndarray
    coef: np.ndarray
    forcing: np.ndarray
    cond_points: np.ndarray
    cond_orders: np.ndarray
    cond_values: np.ndarray
    instances: list = field(default_factory=list)


def linear_batch(cfg: ConfigSpec, seed: int = 0, count: Optional[int] = None,
                 first: int = 0) -> LinearBatch:
    """Instances first..first+count-1 of a linear config, sampled on its grid."""
    count = cfg.batch if count is None else count
    g = grid(cfg)
    lm = equidistant_landmarks(g, cfg.m)
    pts = g[1:]
    p = cfg.order
    coef = np.empty((count, p, pts.size))
    forcing = np.empty((count, pts.size))
    vals = np.empty((count, p))
    insts = []
    for j in range(count):
        inst = _draw_linear(cfg, seed, first + j)
        insts.append(inst)
        coef[j], forcing[j] = inst.sample(pts)
        vals[j] = [c[2] for c in inst.conditions()]
    conds = insts[0].conditions()
    return LinearBatch(cfg, g, lm, pts, coef, forcing,
                       np.array([c[0] for c in conds]),
                       np.array([c[1] for c in conds], dtype=np.int32),
                       vals, insts)


def scaled(cfg: ConfigSpec, **kw) -> ConfigSpec:
    """A copy of cfg with some fields replaced (shrunken parity cases)."""
    d = dict(cfg.__dict__)
    d.update(kw)
    return ConfigSpec(**d)
