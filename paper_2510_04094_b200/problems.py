"""ODE specification types -- the API the hot path consumes.

Field-for-field mirror of the reference's ``pkg/src/nysode/problems.py:22-56``
(``BoundaryCondition``, ``Conditions``, ``LinearOdeSpec``, ``NonlinearOdeSpec``),
so a caller can build specs without the reference installed.  Every solver
entry point duck-types its arguments, so the reference's own spec objects are
accepted unchanged (drop-in).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional


@dataclass(frozen=True)
class BoundaryCondition:
    """y^(order)(point) = value (problems.py:22-28)."""

    point: float
    order: int
    value: float


@dataclass(frozen=True)
class Conditions:
    """kind "ivp" or "bvp" plus the condition entries (problems.py:31-38)."""

    kind: str
    entries: tuple

    def __post_init__(self) -> None:
        if self.kind not in ("ivp", "bvp"):
            raise ValueError(f"unknown condition kind {self.kind!r}")


@dataclass(frozen=True)
class LinearOdeSpec:
    """y^(p) = sum_k f_k(t) y^(p-k) + r(t) (problems.py:41-46)."""

    order: int
    coeffs: tuple
    forcing: Callable
    domain: tuple


@dataclass(frozen=True)
class NonlinearOdeSpec:
    """y^(p) = f(t, y, ..., y^(p-1)) with partials (problems.py:49-56)."""

    order: int
    rhs: Callable
    rhs_partials: tuple
    domain: tuple
    rhs_second_partials: Optional[dict] = None


def ivp(entries) -> Conditions:
    return Conditions("ivp", tuple(BoundaryCondition(*e) for e in entries))
