"""CPU baseline: the oracle restatement of the reference path, timed on the
host's cores (``bench.py`` cpu_baseline / ``--impl reference`` legs only).

The reference (nysode) is pure Python/NumPy and cannot travel to the GPU box,
so the baseline is its restatement (``kind: "port"``), run the way BASELINE.md
§2 prescribes: batched configs use a process pool of N_cores workers with one
BLAS thread each (instances are independent); each worker builds the shared
feature map once and then, per instance, samples the spec callables and runs
``assemble`` + ``solve`` (linear.py:90-158) -- the reference API has no batch
entry, so this is how a reference user solves a shared-grid batch.
"""
from __future__ import annotations

import os
import time

import numpy as np


def _worker_init():
    # forked workers inherit an already-initialised OpenBLAS pool: cap it at
    # runtime (env vars alone would be ignored and oversubscribe the cores)
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    os.environ["OMP_NUM_THREADS"] = "1"
    from threadpoolctl import threadpool_limits

    global _LIMITS
    _LIMITS = threadpool_limits(limits=1)


def _solve_range(args):
    cid, seed, first, count, budget_s, cfg_over = args
    from oracle import nys_port as O
    from paper_2510_04094_b200 import workloads as W

    cfg = W.scaled(W.CONFIGS[cid], **cfg_over) if cfg_over else W.CONFIGS[cid]
    g = W.grid(cfg)
    lm = O.equidistant(g, cfg.m)
    s, v = O.eig_landmarks(cfg.sigma2, lm)
    Wb = O.scaled_basis(s, v)
    t0 = time.perf_counter()
    done = 0
    for i in range(first, first + count):
        inst = W.instance(cid, seed, i, cfg)
        sy = O.assemble(cfg.order, inst.coeff_fns(), inst.forcing_fn, inst.conditions(), g,
                        cfg.gamma, cfg.sigma2, lm, Wb)
        O.solve_kkt(sy["M"], sy["rhs"])
        done += 1
        if budget_s is not None and time.perf_counter() - t0 > budget_s:
            break
    return done, time.perf_counter() - t0


def batch_solves_per_second(cid: int = 2, workers: int | None = None, per_worker: int = 64,
                            budget_s: float | None = None, seed: int = 0, cfg_over=None):
    """Solve a bounded sample of instances on `workers` processes; returns
    (solves/s over the pool's wall time, solved, workers, wall seconds)."""
    import multiprocessing as mp

    workers = workers or os.cpu_count() or 1
    ctx = mp.get_context("fork")
    jobs = [(cid, seed, w * per_worker, per_worker, budget_s, cfg_over) for w in range(workers)]
    t0 = time.perf_counter()
    with ctx.Pool(workers, initializer=_worker_init) as pool:
        res = pool.map(_solve_range, jobs)
    wall = time.perf_counter() - t0
    solved = sum(r[0] for r in res)
    return solved / wall, solved, workers, wall


def single_solve_seconds(cid: int, seed: int = 0, cfg_over=None) -> float:
    """Harness train scope for one linear instance (harness.py:152-163)."""
    from oracle import nys_port as O
    from paper_2510_04094_b200 import workloads as W

    cfg = W.scaled(W.CONFIGS[cid], **cfg_over) if cfg_over else W.CONFIGS[cid]
    g = W.grid(cfg)
    inst = W.instance(cid, seed, 0, cfg)
    t0 = time.perf_counter()
    O.solve_linear_instance(cfg.order, inst.coeff_fns(), inst.forcing_fn, inst.conditions(), g,
                            cfg.gamma, cfg.sigma2, cfg.m)
    return time.perf_counter() - t0
