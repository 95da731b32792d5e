import sys
import numpy as np
sys.path.insert(0, "tests")
from conftest import load_golden
from paper_2510_04094_b200 import newton as NW, nystrom as N, workloads as W
from paper_2510_04094_b200.kernel import RbfKernel
from paper_2510_04094_b200.problems import NonlinearOdeSpec, BoundaryCondition, Conditions
g = load_golden("full_feature_newton")
cfg = W.CONFIGS[3]
grid = g["grid"]
for i in (0, 1):
    inst = W.instance(3, 0, i, cfg)
    spec = NonlinearOdeSpec(1, inst.rhs, (inst.rhs_y,), cfg.domain, {(0, 0): inst.rhs_yy})
    cond = Conditions("ivp", tuple(BoundaryCondition(*c) for c in inst.conditions()))
    for tol in (1e-13, 1e-14, 1e-15, 1e-16, 3e-17):
        N._LARGE_PCHOL_TOL = tol
        fm = N.build_feature_map(RbfKernel(float(g["sigma2"])), grid)
        try:
            model, trace = NW.solve_nonlinear(spec, cond, fm, grid, float(g["gamma"]),
                                              NW.NewtonOptions(max_iters=int(g["max_iters"])))
            st = f"ok its={trace.iterations}"
        except NW.MaxItersExceeded as e:
            model, st = e.model, "maxits"
        except Exception as e:
            print(i, tol, "ERR", type(e).__name__, str(e)[:80]); continue
        y = model.predict(0, grid)
        ref = g[f"i{i}_yhat"]
        print(i, tol, "rank", fm._host["compressed"], "m_eff", fm.m_eff, st,
              "rel vs ref %.2e" % (np.linalg.norm(y - ref) / np.linalg.norm(ref)),
              "err %.2e" % (np.linalg.norm(y - g[f"i{i}_ystar"]) / np.linalg.norm(g[f"i{i}_ystar"])))
