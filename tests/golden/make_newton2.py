"""Golden vectors for the second-order Newton path: the LIVE reference's
``newton.solve_nonlinear`` (p = 2) on workloads.nonlinear2_instance(0, 0..5).

Build container only:  PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_newton2.py
"""
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

from nysode import newton, nystrom  # noqa: E402
from nysode.kernel import RbfKernel  # noqa: E402
from nysode.problems import BoundaryCondition, Conditions, NonlinearOdeSpec  # noqa: E402

from paper_2510_04094_b200 import workloads as W  # noqa: E402


def main(indices=(0, 1, 2, 3, 4, 5)):
    P = W.NONLINEAR2
    g = np.linspace(P["domain"][0], P["domain"][1], P["n"])
    lm = W.equidistant_landmarks(g, P["m"])
    sigma2 = P["sigma"] ** 2
    fmap = nystrom.build_feature_map(RbfKernel(sigma2), lm)
    out = dict(grid=g, landmarks=lm, sigma2=sigma2, gamma=P["gamma"], m_eff=fmap.m_eff,
               eigvals=fmap.eigenvalues, indices=np.array(indices))
    status, yhat, its, err, conds = [], [], [], [], []
    for j, i in enumerate(indices):
        inst = W.nonlinear2_instance(0, i)
        spec = NonlinearOdeSpec(2, inst.rhs, (inst.rhs_y, inst.rhs_yp), inst.domain,
                                inst.second_partials())
        cond = Conditions("ivp", tuple(BoundaryCondition(*c) for c in inst.conditions()))
        t0 = time.perf_counter()
        try:
            mdl, tr = newton.solve_nonlinear(spec, cond, fmap, g, P["gamma"],
                                             newton.NewtonOptions(max_iters=P["newton_max_iters"]))
            st = "converged"
        except newton.MaxItersExceeded as exc:
            mdl, tr, st = exc.model, exc.trace, "max_iters"
        y = mdl.predict(0, g)
        ys = inst.sol(g)
        status.append(st)
        yhat.append(y)
        its.append(tr.iterations)
        err.append(np.linalg.norm(y - ys) / np.linalg.norm(ys))
        conds.append([c[2] for c in inst.conditions()])
        out[f"norms_{j}"] = np.array(tr.residual_norms)
        print(f"  n2[{i}] {inst.kind} k={inst.k:.3f} {st} its={tr.iterations} err={err[-1]:.3e} "
              f"{time.perf_counter() - t0:.2f}s")
    out.update(status=np.array(status), yhat=np.array(yhat), iterations=np.array(its),
               err_vs_exact=np.array(err), cond_values=np.array(conds))
    np.savez_compressed(os.path.join(HERE, "n2_seed0_i0-5.npz"), **out)


if __name__ == "__main__":
    main()
