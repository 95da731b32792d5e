"""solve_many's host side (no GPU): callable sampling on the thread pool raises
the reference's errors (linear.py:104-116) -- non-finite coefficients or
forcing -> FloatingPointError, mixed orders / condition layouts -> ValueError --
before any device work."""
import numpy as np
import pytest

from paper_2510_04094_b200 import batch as BT
from paper_2510_04094_b200 import workloads as W
from paper_2510_04094_b200.problems import BoundaryCondition, Conditions, LinearOdeSpec


def _specs(n, bad=None, what="coef"):
    cfg = W.scaled(W.CONFIGS[2], n=257, batch=n)
    out, conds = [], []
    for b in range(n):
        inst = W.instance(2, 0, b, cfg)
        co, fo = inst.coeff_fns(), inst.forcing_fn
        if b == bad and what == "coef":
            co = (co[0], lambda t: np.full_like(np.asarray(t, float), np.nan))
        if b == bad and what == "forcing":
            fo = lambda t: np.full_like(np.asarray(t, float), np.inf)   # noqa: E731
        out.append(LinearOdeSpec(2, co, fo, inst.domain))
        conds.append(Conditions("ivp", tuple(BoundaryCondition(*c) for c in inst.conditions())))
    return out, conds, W.grid(cfg)


@pytest.mark.parametrize("what", ["coef", "forcing"])
def test_non_finite_samples_raise(what):
    specs, conds, grid = _specs(300, bad=211, what=what)
    with pytest.raises(FloatingPointError):
        BT.solve_many(specs, conds, None, grid, 1e9)


def test_layout_errors():
    specs, conds, grid = _specs(4)
    with pytest.raises(ValueError):
        BT.solve_many(specs, conds[:3], None, grid, 1e9)
    moved = Conditions("ivp", (BoundaryCondition(0.5, 0, 1.0), conds[1].entries[1]))
    with pytest.raises(ValueError):
        BT.solve_many(specs, [conds[0], moved] + conds[2:], None, grid, 1e9)
