"""nysb200 -- B200-native (sm_100a, FP64) hot path of the Nystrom LS-SVM ODE
solver of arXiv 2510.04094 (reference package ``nysode``).

Drop-in modules mirroring the reference API:
``kernel`` (RbfKernel), ``nystrom`` (select_landmarks, build_feature_map,
NystromFeatureMap), ``linear`` (assemble, solve, check_kkt, PrimalModel),
``newton`` (solve_nonlinear), ``problems`` (spec types); plus ``batch`` for
shared-grid batches (config 2) and ``dist`` for multi-GPU sharding.
All numerics run in ``libnysb200.so`` (hand-written CUDA, C ABI in
include/nysb200.h); there is no CPU fallback.
"""
from . import _lib  # noqa: F401

__all__ = ["kernel", "nystrom", "linear", "batch", "problems", "workloads"]
