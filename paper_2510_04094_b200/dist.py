"""Multi-GPU partitioning of the hot path (one process per GPU, torch.distributed).

Two strategies, both from BASELINE.json / SURVEY.md §8(e):

* instance sharding (config 2, batched linear): independent ODEs, rank r owns
  instances [r B/N, (r+1) B/N) -- no collective on the data path
  (:func:`instance_range`).
* row sharding (config 4, one huge ODE): rank r owns a contiguous slab of the
  collocation rows and produces the PARTIAL extended Gram E_r = sum over its
  rows of [D g r]^T [D g r] with the fused kernel (row_begin/row_end of
  ``nys_fused_gram_f64``); one all-reduce(SUM) of the (m_eff+2)^2 doubles
  (528 KB at m = 256) gives every rank the full E, and every rank then solves
  the small KKT system redundantly (no broadcast).  Rows are independent in
  the Gram sum, so this is exact up to summation order (<= 1.5e-14
  on config-4 shapes).  Every rank runs the identical eigensolver, so W is
  bitwise equal across ranks without a broadcast.
"""
from __future__ import annotations

from typing import Optional

import numpy as np

from . import _lib


def instance_range(B: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced instance slab of rank (weak scaling uses B per rank)."""
    base, rem = divmod(B, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def row_ranges(n_rows: int, world: int, align: int = 32) -> list[tuple[int, int]]:
    """Contiguous row slabs, boundaries aligned to the kernel's row tile."""
    tiles = (n_rows + align - 1) // align
    out = []
    for r in range(world):
        lo, hi = instance_range(tiles, world, r)
        out.append((min(lo * align, n_rows), min(hi * align, n_rows)))
    return out


def allreduce_sum(t, group=None):
    """SUM all-reduce of a tensor over the default (or given) process group."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def sharded_gram_ext(fmap, order: int, pts, coef, forcing, rank: int, world: int, group=None):
    """Row-sharded extended Gram: this rank's partial E + one all-reduce.

    pts/coef/forcing are the full (device) sample arrays; only rows of this
    rank's slab are read by the kernel."""
    from .linear import gram_ext_device

    n_c = int(pts.shape[-1]) if hasattr(pts, "shape") else len(pts)
    lo, hi = row_ranges(n_c, world)[rank]
    E = gram_ext_device(fmap, order, pts, coef, forcing, row_begin=lo, row_end=hi)
    return allreduce_sum(E, group)


def solve_row_sharded(fmap, order: int, pts, coef, forcing, cond, gamma: float, rank: int,
                      world: int, group=None):
    """Config-4 solve on `world` GPUs: partial Grams, one all-reduce, redundant
    KKT solve.  Returns the PrimalModel (identical on every rank)."""
    from .linear import AssembledSystem, condition_rows, solve

    E = sharded_gram_ext(fmap, order, pts, coef, forcing, rank, world, group)
    Ac, beta, vals = condition_rows(cond, fmap)
    host_pts = pts.cpu().numpy() if hasattr(pts, "cpu") else np.asarray(pts)
    sy = AssembledSystem(constraint_points=host_pts, gamma=float(gamma), g=None, r=None,
                         coeff_values=None, cond_rows=Ac.reshape(len(cond.entries), -1),
                         cond_bias=beta, cond_values=vals, fmap=fmap, order=order, d_gram=E)
    return solve(sy, fmap)
