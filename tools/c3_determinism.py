"""Run the config-3 Newton ladder three times; report bitwise agreement."""
import os
import sys

sys.path.insert(0, os.environ.get("NYS_PKG_ROOT") or
                os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
if os.environ.get("NYS_PROBE_LIB"):
    from paper_2510_04094_b200 import _lib
    _lib.load(os.environ["NYS_PROBE_LIB"])

from paper_2510_04094_b200 import newton as NW, nystrom as N, workloads as W
from paper_2510_04094_b200.kernel import RbfKernel
from paper_2510_04094_b200.problems import ivp

cfg = W.CONFIGS[3]
B = cfg.batch
g = W.grid(cfg)
lm = W.equidistant_landmarks(g, cfg.m)
insts = [W.instance(3, 0, i) for i in range(B)]
pts = g[1:]
fam = NW.SeparableFamily(np.stack([i.g_fn(pts) for i in insts]),
                         np.array([i.quad_coeff for i in insts]),
                         np.array([i.sin_coeff for i in insts]))
vals = np.array([[i.conditions()[0][2]] for i in insts])
cond = ivp([(0.0, 0, 0.0)])
res = []
for rep in range(3):
    fm = N.build_feature_map(RbfKernel(cfg.sigma2), lm)
    eng = NW.NewtonBatch(fm, g, cond, vals, cfg.gamma, family=fam)
    st, X, tr, rung = eng.solve(max_iters=cfg.newton_max_iters)
    res.append((st, X, rung, fm.eigenvalues.copy()))
    print(rep, np.bincount(st, minlength=4), np.bincount(rung))
for r in (1, 2):
    print("run", r, "vs 0: eig equal", np.array_equal(res[r][3], res[0][3]),
          "status equal", np.array_equal(res[r][0], res[0][0]),
          "X equal", np.array_equal(res[r][1], res[0][1], equal_nan=True),
          "rows differing", int((~np.all((res[r][1] == res[0][1]) | (np.isnan(res[r][1]) & np.isnan(res[0][1])), axis=1)).sum()))
