"""Config-3 census: run the LIVE reference (``nysode``) on all 256 bench
instances (seed 0) and store each outcome -- status, iteration count, the
solution vector x and its error vs the manufactured solution -- plus the
reference's landmark eigenpairs (x is expressed in that basis).  A second pass
re-runs the reference with only its landmark eigensolver driver swapped
(scipy's dsyev for numpy's dsyevd) and stores that outcome as status_dsyev /
iterations_dsyev, and three more passes with the landmark matrix perturbed by
at most one ulp per entry (seeded) store status_perturbed: the reference's own
outcome sensitivity to rounding-level noise, the yardstick of the GPU census
test.

Build container only (``/root/reference`` is absent on the GPU box):
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_c3_census.py
Parallel over instances (one BLAS thread per worker process).
"""
from __future__ import annotations

import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))


def _init():
    os.environ["OMP_NUM_THREADS"] = "1"
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    sys.path.insert(0, REF)
    sys.path.insert(0, ROOT)
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)


def _solve_dsyev(i):
    import scipy.linalg as sl

    np.linalg.eigh = lambda A: sl.eigh(A, driver="ev")   # worker process only
    return _solve(i)


def _solve_perturbed(args):
    """The reference on its landmark matrix with every entry moved by at most
    one ulp (symmetric, seeded): rounding-level input noise."""
    i, seed = args
    orig = np.linalg.eigh

    def eigh(A):
        rng = np.random.default_rng(seed)
        U = np.triu(rng.integers(-1, 2, size=A.shape).astype(float))
        U = U + np.triu(U, 1).T
        return orig(A * (1.0 + np.finfo(float).eps * U))

    np.linalg.eigh = eigh
    try:
        return _solve(i)
    finally:
        np.linalg.eigh = orig


def _solve(i):
    from nysode import newton, nystrom
    from nysode.kernel import RbfKernel
    from nysode.problems import BoundaryCondition, Conditions, NonlinearOdeSpec

    from paper_2510_04094_b200 import workloads as W
    cfg = W.CONFIGS[3]
    g = W.grid(cfg)
    lm = W.equidistant_landmarks(g, cfg.m)
    fmap = nystrom.build_feature_map(RbfKernel(cfg.sigma2), lm)
    inst = W.instance(3, 0, i, cfg)
    spec = NonlinearOdeSpec(1, inst.rhs, (inst.rhs_y,), cfg.domain, {(0, 0): inst.rhs_yy})
    cond = Conditions("ivp", tuple(BoundaryCondition(*c) for c in inst.conditions()))
    opts = newton.NewtonOptions(max_iters=cfg.newton_max_iters)
    try:
        mdl, tr = newton.solve_nonlinear(spec, cond, fmap, g, cfg.gamma, opts)
        status = 0
    except newton.MaxItersExceeded as exc:      # harness.py:173-175
        mdl, tr = exc.model, exc.trace
        status = 1
    except newton.DivergenceError:
        return i, 2, 0, None, np.nan
    except newton.SingularJacobianError:
        return i, 3, 0, None, np.nan
    y = mdl.predict(0, g)
    ys = inst.sol(g)
    x = np.concatenate([mdl.omega, [mdl.bias], mdl.multipliers])
    return i, status, tr.iterations, x, float(np.linalg.norm(y - ys) / np.linalg.norm(ys))


PERTURB_SEEDS = (1, 2, 3)


def main():
    t0 = time.time()
    n = 256
    with ProcessPoolExecutor(max_workers=os.cpu_count(), initializer=_init) as ex:
        res = sorted(ex.map(_solve, range(n)))
    with ProcessPoolExecutor(max_workers=os.cpu_count(), initializer=_init) as ex:
        res_ev = sorted(ex.map(_solve_dsyev, range(n)))
    res_pert = []
    for seed in PERTURB_SEEDS:
        with ProcessPoolExecutor(max_workers=os.cpu_count(), initializer=_init) as ex:
            res_pert.append(sorted(ex.map(_solve_perturbed, [(i, seed) for i in range(n)])))
    me = next(r[3].size for r in res if r[3] is not None)
    X = np.full((n, me), np.nan)
    for i, st, its, x, err in res:
        if x is not None:
            X[i] = x
    _init()
    from nysode import nystrom
    from nysode.kernel import RbfKernel

    from paper_2510_04094_b200 import workloads as W
    cfg = W.CONFIGS[3]
    fmap = nystrom.build_feature_map(RbfKernel(cfg.sigma2),
                                     W.equidistant_landmarks(W.grid(cfg), cfg.m))
    np.savez_compressed(os.path.join(HERE, "c3_census_seed0.npz"),
                        eigvals=fmap.eigenvalues, eigvecs=fmap.eigenvectors,
                        status=np.array([r[1] for r in res], np.int32),
                        iterations=np.array([r[2] for r in res], np.int32),
                        x=X, err_vs_exact=np.array([r[4] for r in res]),
                        status_dsyev=np.array([r[1] for r in res_ev], np.int32),
                        iterations_dsyev=np.array([r[2] for r in res_ev], np.int32),
                        status_perturbed=np.array([[r[1] for r in rp] for rp in res_pert],
                                                  np.int32))
    st = np.bincount([r[1] for r in res], minlength=4)
    st_ev = np.bincount([r[1] for r in res_ev], minlength=4)
    print(f"c3 census: status counts {st.tolist()} (dsyev driver {st_ev.tolist()}) "
          f"in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
