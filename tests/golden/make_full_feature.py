"""Golden vectors for the m = n full-feature comparator: the LIVE reference's
``baselines.full_feature_baseline`` (baselines.py:170-194) on linear catalog
problems, sampled on the constraint points (no reference code is stored), plus
the same run with LAPACK's dsyev driver in place of dsyevd as the reference's
own eigensolver sensitivity (the parity yardstick).

Build container only:  PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_full_feature.py
"""
import os
import sys

import numpy as np
import scipy.linalg as sl

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

from nysode import baselines, linear, nystrom, problems  # noqa: E402

PIDS = (1, 7, 8, 12, 16)


def main():
    out = {}
    orig = np.linalg.eigh
    for pid in PIDS:
        p = problems.get_problem(pid)
        d = p.defaults
        g = problems.grid_for(p, d.n)
        mdl, secs = baselines.full_feature_baseline(p, d.gamma, d.sigma2, d.n)
        nystrom.np.linalg.eigh = lambda A: sl.eigh(A, driver="ev")
        try:
            mdl2, _ = baselines.full_feature_baseline(p, d.gamma, d.sigma2, d.n)
        finally:
            nystrom.np.linalg.eigh = orig
        pts = linear.constraint_points(p.conditions, g)
        coef = np.stack([np.broadcast_to(np.asarray(f(pts), dtype=float), pts.shape)
                         for f in p.spec.coeffs])
        forcing = np.broadcast_to(np.asarray(p.spec.forcing(pts), dtype=float), pts.shape)
        ents = p.conditions.entries
        key = f"p{pid}"
        out.update({
            f"{key}_kind": np.array(p.conditions.kind), f"{key}_order": np.array(p.spec.order),
            f"{key}_gamma": np.array(d.gamma), f"{key}_sigma2": np.array(d.sigma2),
            f"{key}_n": np.array(d.n), f"{key}_lo": np.array(p.domain[0]),
            f"{key}_hi": np.array(p.domain[1]), f"{key}_pts": pts, f"{key}_coef": coef,
            f"{key}_forcing": np.array(forcing),
            f"{key}_cond_points": np.array([bc.point for bc in ents], dtype=float),
            f"{key}_cond_orders": np.array([bc.order for bc in ents], dtype=int),
            f"{key}_cond_values": np.array([bc.value for bc in ents], dtype=float),
            f"{key}_yhat": mdl.predict(0, g), f"{key}_yhat_dsyev": mdl2.predict(0, g),
            f"{key}_yhat1": mdl.predict(1, g),
            f"{key}_m_eff": np.array(mdl.feature_map.m_eff),
            f"{key}_m_eff_dsyev": np.array(mdl2.feature_map.m_eff),
            f"{key}_eigvals": mdl.feature_map.eigenvalues, f"{key}_seconds": np.array(secs),
        })
        ss = np.linalg.norm(mdl2.predict(0, g) - mdl.predict(0, g)) / np.linalg.norm(mdl.predict(0, g))
        print(f"P{pid}: m_eff {mdl.feature_map.m_eff} self-sens {ss:.2e} {secs:.3f}s")
    out["pids"] = np.array(PIDS)
    np.savez_compressed(os.path.join(HERE, "full_feature.npz"), **out)


if __name__ == "__main__":
    main()


def main_newton(indices=(0, 1)):
    """Full-feature Newton (the nonlinear branch of baselines.py:186-191) on
    config-3 instances, whose callables live in this package's workloads."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    from nysode import newton
    from nysode.kernel import RbfKernel
    from nysode.problems import BoundaryCondition, Conditions, NonlinearOdeSpec
    from paper_2510_04094_b200 import workloads as W
    cfg = W.CONFIGS[3]
    g = W.grid(cfg)
    out = dict(grid=g, sigma2=cfg.sigma2, gamma=cfg.gamma, max_iters=cfg.newton_max_iters,
               indices=np.array(indices))
    orig = np.linalg.eigh
    for i in indices:
        inst = W.instance(3, 0, i, cfg)
        spec = NonlinearOdeSpec(1, inst.rhs, (inst.rhs_y,), cfg.domain, {(0, 0): inst.rhs_yy})
        cond = Conditions("ivp", tuple(BoundaryCondition(*c) for c in inst.conditions()))
        res = []
        for drv in ("evd", "ev"):
            if drv == "ev":
                nystrom.np.linalg.eigh = lambda A: sl.eigh(A, driver="ev")
            try:
                fm = nystrom.build_feature_map(RbfKernel(cfg.sigma2), g)
                try:
                    mdl, tr = newton.solve_nonlinear(spec, cond, fm, g, cfg.gamma,
                                                     newton.NewtonOptions(max_iters=cfg.newton_max_iters))
                    st = "converged"
                except newton.MaxItersExceeded as exc:
                    mdl, tr, st = exc.model, exc.trace, "max_iters"
            finally:
                nystrom.np.linalg.eigh = orig
            res.append((mdl.predict(0, g), st, fm.m_eff, tr.iterations))
        out[f"i{i}_yhat"], out[f"i{i}_status"], out[f"i{i}_m_eff"], out[f"i{i}_its"] = res[0]
        out[f"i{i}_yhat_dsyev"] = res[1][0]
        out[f"i{i}_status_dsyev"] = res[1][1]
        out[f"i{i}_ystar"] = inst.sol(g)
        ss = np.linalg.norm(res[1][0] - res[0][0]) / np.linalg.norm(res[0][0])
        print(f"c3[{i}] full-feature: {res[0][1]} its={res[0][3]} m_eff={res[0][2]} self-sens {ss:.2e}")
    np.savez_compressed(os.path.join(HERE, "full_feature_newton.npz"), **out)


if __name__ == "__main__" and os.environ.get("NYS_FF_NEWTON"):
    main_newton()
