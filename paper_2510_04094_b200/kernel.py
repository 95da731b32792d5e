"""RBF kernel parameters (mirror of ``pkg/src/nysode/kernel.py:47-59``).

The kernel values themselves are only ever generated inside the CUDA kernels
(csrc/common.cuh: ``nys::Hermite`` + ``nys::rbf``), never on the host.
"""
from __future__ import annotations

from dataclasses import dataclass

from ._refcompat import ref_base

MAX_DERIV_ORDER = 4          # kernel.py:19


class UnsupportedOrderError(*ref_base("kernel", "UnsupportedOrderError", ValueError)):
    """Derivative order outside 0..4 (kernel.py:22-23)."""


@dataclass(frozen=True)
class RbfKernel:
    """K(u, v) = exp(-(u - v)^2 / sigma2) (kernel.py:47-55)."""

    sigma2: float

    def __post_init__(self) -> None:
        if not self.sigma2 > 0:
            raise ValueError(f"sigma2 must be positive, got {self.sigma2}")


def check_order(a: int) -> None:
    if not 0 <= a <= MAX_DERIV_ORDER:
        raise UnsupportedOrderError(
            f"derivative order {a} not supported (must be 0..{MAX_DERIV_ORDER})")
