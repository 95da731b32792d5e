"""CPU baseline: the oracle restatement of the reference path, timed on the
host's cores (``bench.py`` cpu_baseline / ``--impl reference`` legs only).

TEST / BASELINE INFRASTRUCTURE ONLY.  The reference (nysode) is pure
Python/NumPy and cannot travel to the GPU box, so the baseline is its
restatement (``kind: "port"``), run the way BASELINE.md §2 prescribes:

* batched configs (2, 3): a process pool of N_cores workers with one BLAS
  thread each (instances are independent); each worker builds the shared
  feature map once and then, per instance, runs the reference's per-spec
  entry points (linear.assemble + linear.solve, or newton.solve_nonlinear with
  max_iters = 20) on the spec CALLABLES, exactly as a reference user would;
* single-instance configs (0, 1, 4): one process, all BLAS threads.
  Config 4 needs ~42 GB and ~135 s per solve on the reference; the bounded
  sample assembles a row slab with the reference's own per-order feature
  matrices and the O(n) assembly cost is scaled to the full n (stated in the
  sample string).
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


def _cfg(cid, cfg_over):
    from paper_2510_04094_b200 import workloads as W

    return W.scaled(W.CONFIGS[cid], **cfg_over) if cfg_over else W.CONFIGS[cid]


def _solve_range(args):
    cid, seed, first, count, budget_s, cfg_over = args
    from oracle import newton_port as NP
    from oracle import nys_port as O
    from paper_2510_04094_b200 import workloads as W

    cfg = _cfg(cid, cfg_over)
    g = W.grid(cfg)
    lm = O.equidistant(g, cfg.m)
    s, v = O.eig_landmarks(cfg.sigma2, lm)
    Wb = O.scaled_basis(s, v)
    t0 = time.perf_counter()
    done = 0
    for i in range(first, first + count):
        inst = W.instance(cid, seed, i, cfg)
        if cfg.nonlinear:
            spec = NP.NlSpec(1, inst.rhs, (inst.rhs_y,), {(0, 0): inst.rhs_yy})
            try:
                NP.solve_nonlinear(spec, inst.conditions(), g, cfg.gamma, cfg.sigma2, lm, Wb,
                                   max_iters=cfg.newton_max_iters)
            except (NP.MaxIters, NP.Divergence, NP.SingularJac):
                pass                      # the harness records the outcome; still one solve
        else:
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


def single_solve_seconds(cid: int, seed: int = 0, cfg_over=None, reps: int = 3) -> float:
    """Harness train scope for one linear instance (harness.py:152-163), best of reps."""
    from oracle import nys_port as O
    from paper_2510_04094_b200 import workloads as W

    cfg = _cfg(cid, cfg_over)
    g = W.grid(cfg)
    inst = W.instance(cid, seed, 0, cfg)
    best = float("inf")
    for _ in range(reps):
        t0 = time.perf_counter()
        O.solve_linear_instance(cfg.order, inst.coeff_fns(), inst.forcing_fn, inst.conditions(), g,
                                cfg.gamma, cfg.sigma2, cfg.m)
        best = min(best, time.perf_counter() - t0)
    return best


def c4_solve_seconds_estimate(sample_rows: int = 1 << 18, seed: int = 0):
    """Config 4 on the reference path, bounded: eigendecomposition + KKT solve
    timed in full; assembly timed on `sample_rows` constraint rows (the
    reference's per-order feature_matrix + combine + D^T D, linear.py:103-133)
    and scaled by n_c / sample_rows (assembly is O(n) in rows)."""
    from oracle import nys_port as O
    from paper_2510_04094_b200 import workloads as W

    cfg = W.CONFIGS[4]
    g = W.grid(cfg)
    inst = W.instance(4, seed, 0, cfg)
    t0 = time.perf_counter()
    lm = O.equidistant(g, cfg.m)
    s, v = O.eig_landmarks(cfg.sigma2, lm)
    Wb = O.scaled_basis(s, v)
    t_eig = time.perf_counter() - t0
    sub = np.concatenate([g[:1], g[1:1 + sample_rows]])
    t0 = time.perf_counter()
    sy = O.assemble(cfg.order, inst.coeff_fns(), inst.forcing_fn, inst.conditions(), sub,
                    cfg.gamma, cfg.sigma2, lm, Wb)
    t_asm = time.perf_counter() - t0
    t0 = time.perf_counter()
    O.solve_kkt(sy["M"], sy["rhs"])
    t_solve = time.perf_counter() - t0
    scale = (g.size - 1) / sample_rows
    return t_eig + t_asm * scale + t_solve, dict(t_eig=t_eig, t_asm_sample=t_asm, scale=scale,
                                                 t_solve=t_solve)


def _yhat_range(args):
    cid, seed, indices, cfg_over = args
    from oracle import nys_port as O
    from paper_2510_04094_b200 import workloads as W

    cfg = _cfg(cid, cfg_over)
    g = W.grid(cfg)
    lm = O.equidistant(g, cfg.m)
    s, v = O.eig_landmarks(cfg.sigma2, lm)
    Wb = O.scaled_basis(s, v)
    me = Wb.shape[1]
    out = []
    for i in indices:
        inst = W.instance(cid, seed, i, cfg)
        sy = O.assemble(cfg.order, inst.coeff_fns(), inst.forcing_fn, inst.conditions(), g,
                        cfg.gamma, cfg.sigma2, lm, Wb)
        x = O.solve_kkt(sy["M"], sy["rhs"])
        y = O.predict(cfg.sigma2, lm, Wb, x[:me], float(x[me]), 0, g)
        ys = inst.sol(g)
        out.append((i, y, float(np.linalg.norm(y - ys) / np.linalg.norm(ys))))
    return out


def reference_yhat(cid: int, indices, workers: int | None = None, seed: int = 0,
                   cfg_over=None) -> dict:
    """Oracle y_hat on the grid (and its error vs y*) for the given linear
    instances -- the checker bench.py runs beside its cpu_baseline leg to
    compare the timed batch's solutions with (never the thing measured)."""
    import multiprocessing as mp

    indices = list(indices)
    workers = max(1, min(workers or os.cpu_count() or 1, len(indices)))
    parts = [indices[w::workers] for w in range(workers)]
    ctx = mp.get_context("fork")
    with ctx.Pool(workers, initializer=_worker_init) as pool:
        res = pool.map(_yhat_range, [(cid, seed, p, cfg_over) for p in parts if p])
    return {i: (y, e) for part in res for i, y, e in part}
