"""The m = n full-feature comparator on the device.

Mirror of ``baselines.full_feature_baseline`` (pkg/src/nysode/baselines.py:170-194):
the same pipeline with every grid point as a landmark.  The problem argument is
duck-typed like the reference's ``BenchmarkProblem`` (``domain``, ``spec``,
``conditions``, ``is_linear``, ``defaults.newton_iters``), so the reference's
catalog objects work unchanged.  The m x m landmark eigendecomposition runs on
the compressed large-m path of :func:`nystrom.build_feature_map` and the
assembly on explicit feature matrices (:func:`linear.gram_ext_device`).
"""
from __future__ import annotations

import time

import numpy as np

from . import linear, newton, nystrom
from ._refcompat import ref_base
from .kernel import RbfKernel

FULL_FEATURE_MAX_N = 5000       # baselines.py:167


class MemoryGuardError(*ref_base("baselines", "MemoryGuardError", ValueError)):
    """n above the full-feature cap (baselines.py:170-171)."""


def grid_for(problem, n: int) -> np.ndarray:
    """problems.grid_for (problems.py:98-100)."""
    t1, tn = problem.domain
    return np.linspace(t1, tn, n)


def full_feature_baseline(problem, gamma: float, sigma2: float, n: int,
                          drop_tol: float = nystrom.DEFAULT_DROP_TOL):
    """Same pipeline with landmarks = entire grid; returns (model, train_seconds)."""
    if n > FULL_FEATURE_MAX_N:
        raise MemoryGuardError(f"full-feature baseline capped at n={FULL_FEATURE_MAX_N}")
    grid = grid_for(problem, n)
    k = RbfKernel(sigma2=sigma2)
    t0 = time.perf_counter()
    fmap = nystrom.build_feature_map(k, grid, drop_tol=drop_tol)
    if problem.is_linear:
        system = linear.assemble(problem.spec, problem.conditions, fmap, grid, gamma)
        model = linear.solve(system, fmap)
    else:
        iters = problem.defaults.newton_iters or 100
        model, _ = newton.solve_nonlinear(problem.spec, problem.conditions, fmap, grid, gamma,
                                          newton.NewtonOptions(max_iters=iters))
    train_seconds = time.perf_counter() - t0
    return model, train_seconds
