"""Trace the gamma-continuation rung (newton.py:352-373) of one config-3
instance on the device, stage by stage (compare with the reference's)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2510_04094_b200 import newton as NW, nystrom as N, workloads as W
from paper_2510_04094_b200.kernel import RbfKernel
from paper_2510_04094_b200.problems import ivp

cfg = W.CONFIGS[3]
g = W.grid(cfg)
lm = W.equidistant_landmarks(g, cfg.m)
fm = N.build_feature_map(RbfKernel(cfg.sigma2), lm)
for i in [int(a) for a in sys.argv[1:]]:
    inst = W.instance(3, 0, i)
    pts = g[1:]
    fam = NW.SeparableFamily(inst.g_fn(pts)[None], np.array([inst.quad_coeff]),
                             np.array([inst.sin_coeff]))
    eng = NW.NewtonBatch(fm, g, ivp([(0.0, 0, 0.0)]), np.array([[inst.conditions()[0][2]]]),
                         cfg.gamma, family=fam)
    x = eng.const_state([0])
    for gm in (1e0, 1e2, 1e4):
        st, Xn, tr = eng.solve_once([0], x, gm, 1e-8 * (1 + gm), True, cfg.newton_max_iters)
        print(f"{i} stage {gm:g}: st={st[0]} its={len(tr[0]) - 1} norms="
              f"{['%.3e' % v for v in tr[0][:6]]} ... {tr[0][-1]:.3e}")
        print("   omega[:3]", Xn[0, :3], "bias", Xn[0, eng.me])
        x = eng.model_state([0], Xn[:1])
    st, Xn, tr = eng.solve_once([0], x, cfg.gamma, 1e-10 * (1 + cfg.gamma), True,
                                cfg.newton_max_iters)
    print(f"{i} final: st={st[0]} its={len(tr[0]) - 1} norms={['%.3e' % v for v in tr[0]]}")
